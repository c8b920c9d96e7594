#!/usr/bin/env python
"""Summarise an `ncu --set full` raw CSV (ncu -i X.ncu-rep --page raw --csv) into one line
per kernel (duration, DRAM bytes, tensor-pipe activity, occupancy, top stall reasons) and
write the per-launch DRAM traffic bench.py reports as roofline.traffic.
  python tools/ncu_summary.py profiles/rNN_ncu_full_raw.csv profiles/rNN_ncu_full_summary.txt
"""
import csv
import json
import os
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "launch__grid_size"]
# bench.py phase name for each kernel (the dominant kernel's traffic is reported per launch)
PHASE = {"sparse_adam": "sparse_adam", "gather_instances": "gather_instances",
         "gemm_ts_kernel<0": "tower_gemm1", "gemm_ts_kernel<1": "tower_gemm3",
         "gemm_dx_persistent": "tower_gemm2", "zero_rows_b": "zero_grads",
         "vsi_first": "vsi_first", "admit_kernel": "admit", "owner_reduce": "owner_reduce"}


def to_bytes(v, unit):
    f = float(v.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    stall_cols = [h for h in hdr if h.startswith("smsp__average_warp_latency_issue_stalled")
                  or (h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued"))]
    out, traffic = [], {}
    for r in rows[2:]:
        name = r[idx["Kernel Name"]]
        vals = {}
        for k in KEYS:
            if k in idx:
                vals[k] = r[idx[k]]
        rd = to_bytes(vals.get("dram__bytes_read.sum", "0"), units[idx["dram__bytes_read.sum"]])
        wr = to_bytes(vals.get("dram__bytes_write.sum", "0"), units[idx["dram__bytes_write.sum"]])
        st = sorted(((float(r[idx[h]].replace(",", "") or 0), h.split("stalled_")[-1]) for h in stall_cols
                     if r[idx[h]] not in ("", "n/a")), reverse=True)[:6]
        out.append(f"{name[:70]} | time_ns={vals.get('gpu__time_duration.sum')} | dram_read_MB={rd/1e6:.2f}"
                   f" | dram_write_MB={wr/1e6:.2f} | tensor_active%={vals.get(KEYS[3])}"
                   f" | warps_active%={vals.get(KEYS[4])} | l2%={vals.get(KEYS[5])}"
                   f" | regs={vals.get(KEYS[6])} | grid={vals.get(KEYS[7])}\n   stalls: "
                   + ", ".join(f"{n}={v:.2f}" for v, n in st))
        for pat, ph in PHASE.items():
            if pat in name:
                traffic[ph] = int(rd + wr)
    open(dst, "w").write("\n".join(out) + "\n")
    tj = os.path.join(os.path.dirname(dst), "ncu_traffic.json")
    json.dump({"source": os.path.basename(src),
               "note": "ncu --set full (cold L2 per replay): dram__bytes_read.sum + "
                       "dram__bytes_write.sum per launch", "dram_bytes_per_launch": traffic},
              open(tj, "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
