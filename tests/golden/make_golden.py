"""Regenerates tests/golden/golden.json from the REFERENCE's own compiled code.

Run in the build container (where /root/reference exists):
    make -C oracle && python tests/golden/make_golden.py

Everything here comes from oracle/_ref/libsfctr_ref.so, i.e. the reference's
present translation units (proj/core/src/{generator,vsi,host_store,
cache_buffer,config}.cpp + rng.hpp/comm.hpp) driven through oracle/ref_shim.cpp,
plus the SPEC.md worked examples. Large arrays are stored as sha256 digests of
their little-endian bytes. The GPU box never runs this script; it only reads
the committed JSON.
"""
import hashlib
import json
import os
import struct
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import ref, ref_generate, ref_vsi  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).view(np.uint8).tobytes())
    return h.hexdigest()


def dhex(x):
    return struct.pack("<d", float(x)).hex()


def main():
    R = ref()
    out = {"source": "oracle/_ref/libsfctr_ref.so (reference TUs @ /root/reference/proj/core)"}

    # rng.hpp:27-56
    out["fnv1a64"] = {s: format(R.ref_fnv1a64(s.encode(), len(s)), "016x")
                      for s in ["", "a", "68fd1e64", "embed", "batch", "truth"]}
    out["derive_seed"] = [[b, lbl, i, format(R.ref_derive_seed(b, lbl.encode(), i), "016x")]
                          for b in (0, 7, 12345) for lbl in ("batch", "embed", "truth")
                          for i in (0, 1, 33799999)]
    # generator.cpp:77-80,110-115
    emb = {}
    for f in (0, 1, 17, 999999, 33799999, 999999999):
        v = np.zeros(80)
        R.ref_initial_embedding(7, f, 80, v)
        emb[str(f)] = [dhex(x) for x in v]
    out["initial_embedding_seed7_d80"] = emb
    out["truth_weight_seed7"] = {str(f): dhex(R.ref_truth_weight(7, f)) for f in (0, 1, 5, 12345)}
    # comm.hpp:36-41 (+SPEC.md:60-62)
    out["allreduce_bytes"] = [[p, w, R.ref_allreduce_bytes(p, w)]
                              for p, w in [(1000, 1), (1000, 2), (1024, 4), (1000, 3), (0, 8),
                                           (26572800, 8), (7, 7)]]

    # generator.cpp:82-108 + vsi.cpp:23-54 on the BASELINE configs
    gens = []
    cases = [
        # name, workers, fields, batch_per_worker, vocab, seed, zipf, steps
        ("tiny", 2, 3, 4, 50, 7, 1.2, [0, 1]),
        ("cfg1", 1, 26, 1024, 1_000_000, 7, 1.2, [0, 1, 2]),
        ("cfg1_s105", 1, 26, 1024, 1_000_000, 7, 1.05, [0]),
        ("mini_w4", 4, 26, 256, 100_000, 7, 1.2, [0, 1, 5]),
        ("cfg2_w1", 1, 39, 8192, 33_800_000, 7, 1.05, [0]),
        ("cfg2_w2", 2, 39, 8192, 33_800_000, 7, 1.05, [0]),
        ("cfg2_w4", 4, 39, 8192, 33_800_000, 7, 1.05, [0]),
        ("cfg2_w8", 8, 39, 8192, 33_800_000, 7, 1.05, [0]),
        ("cfg3_s2", 8, 26, 1024, 1_000_000, 7, 2.0, [0]),
    ]
    for name, W, F, b, vocab, seed, zipf, steps in cases:
        for step in steps:
            f, y = ref_generate(W, F, b, vocab, seed, zipf, step)
            rows = W * b
            gids, vids, rr = ref_vsi(f, y, rows, F, W)
            rec = {"name": name, "workers": W, "fields": F, "batch": b, "vocab": vocab,
                   "seed": seed, "zipf": zipf, "step": step,
                   "features_sha256": sha(f), "labels_sha256": sha(y),
                   "positives": int(y.sum()), "unique": int(len(gids)),
                   "global_ids_sha256": sha(gids), "virtual_ids_sha256": sha(vids),
                   "row_ranges": rr.tolist()}
            if rows * F <= 64:
                rec["features"] = f.tolist()
                rec["labels"] = y.tolist()
                rec["global_ids"] = gids.tolist()
                rec["virtual_ids"] = vids.tolist()
            gens.append(rec)
            print(name, step, len(gids), file=sys.stderr)
    out["batches"] = gens

    # vsi.cpp on the SPEC.md:132-134 examples
    vsi_ex = []
    for rows, F, feats in [(2, 3, [1, 3, 2, 2, 3, 1]), (1, 1, [5]), (2, 2, [2, 2, 2, 2])]:
        g, v, _ = ref_vsi(np.array(feats, np.uint64), np.zeros(rows, np.uint8), rows, F, 1)
        vsi_ex.append({"rows": rows, "fields": F, "features": feats, "global_ids": g.tolist(),
                       "virtual_ids": v.tolist()})
    out["vsi_examples"] = vsi_ex
    # vsi.cpp on arbitrary u64 FeatureIds (ids >= 2^32, the all-ones id, repeats)
    rng = np.random.default_rng(2026)
    u64_ex = []
    for rows, F in [(64, 8), (512, 26)]:
        pool = np.concatenate([rng.integers(0, 1 << 62, 40, dtype=np.uint64) * np.uint64(3),
                               np.array([0, 1, (1 << 32) - 1, 1 << 32, (1 << 64) - 1,
                                         (1 << 64) - 2], np.uint64)])
        f = pool[rng.integers(0, pool.size, rows * F)]
        g, v, _ = ref_vsi(f, np.zeros(rows, np.uint8), rows, F, 1)
        rec = {"rows": rows, "fields": F, "features_sha256": sha(f), "unique": int(len(g)),
               "global_ids_sha256": sha(g), "virtual_ids_sha256": sha(v)}
        if rows * F <= 512:  # the larger batch is regenerated by the tests (same rng calls)
            rec["features"] = [str(int(x)) for x in f]
        u64_ex.append(rec)
    out["vsi_u64_examples"] = u64_ex

    # CacheBuffer (cache_buffer.cpp) + HostStore (host_store.cpp): a seeded
    # random admit/evict/touch trace; records every returned slot and the final table.
    rng = np.random.default_rng(1234)
    cap, dim = 16, 4
    c = R.ref_cache_create(7, dim, cap)
    resident = []
    ops = []
    step = 0
    for _ in range(400):
        step += 1
        r = rng.random()
        if (r < 0.55 and len(resident) < cap) or not resident:
            f = int(rng.integers(0, 64))
            if f in resident:
                R.ref_cache_touch(c, f, step)
                ops.append(["touch", f, step])
                continue
            s = R.ref_cache_admit(c, f, step)
            resident.append(f)
            ops.append(["admit", f, step, int(s)])
        else:
            f = resident.pop(int(rng.integers(0, len(resident))))
            R.ref_cache_set_needed_soon(c, f, 0)
            rc = R.ref_cache_evict(c, f)
            ops.append(["evict", f, step, int(rc)])
    feat = np.zeros(cap, np.uint64)
    lu = np.zeros(cap, np.int64)
    seq = np.zeros(cap, np.uint64)
    R.ref_cache_slots(c, feat, lu, seq)
    out["cache_trace"] = {"capacity": cap, "dim": dim, "seed": 7, "ops": ops,
                          "final_features": [int(x) if x != 2**64 - 1 else -1 for x in feat],
                          "final_last_use": lu.tolist(), "final_admit_seq": seq.tolist(),
                          "host_size": int(R.ref_cache_host_size(c))}
    # eviction-safety asserts (cache_buffer.cpp:59-60) — status 3 = LogicError
    c2 = R.ref_cache_create(7, dim, 4)
    R.ref_cache_admit(c2, 10, 0)
    R.ref_cache_admit(c2, 20, 0)
    needed_soon_rc = R.ref_cache_evict(c2, 10)  # admitted => needed_soon
    R.ref_cache_set_needed_soon(c2, 20, 0)
    R.ref_cache_pin(c2, 20, 1)
    pinned_rc = R.ref_cache_evict(c2, 20)
    out["eviction_safety"] = {"needed_soon_status": needed_soon_rc, "pinned_status": pinned_rc}
    R.ref_cache_destroy(c)
    R.ref_cache_destroy(c2)

    # config.cpp validation statuses (1 = ConfigError)
    out["config_checks"] = [[k, v, R.ref_config_check(k.encode(), v.encode(), 1)]
                            for k, v in [("workers", "8"), ("workers", "0"), ("dim", "-3"),
                                         ("zipf", "abc"), ("bogus", "1"), ("vocab", "33800000"),
                                         ("beta1", "1.0"), ("lookahead", "2"),
                                         ("data", "synthetic"), ("data", "criteo:/tmp/day_0.tsv"),
                                         ("data", "criteo:"), ("data", "parquet:/x")]]

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", os.path.join(HERE, "golden.json"), file=sys.stderr)


if __name__ == "__main__":
    main()
