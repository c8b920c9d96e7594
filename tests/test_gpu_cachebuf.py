"""The standalone device CacheBuffer / HostStore / manager (sfctr_cache_*) against the
reference's own CacheBuffer + HostStore (oracle/_ref, compiled from cache_buffer.cpp /
host_store.cpp) and its committed golden trace; the manager step against the SPEC.md:195
worked example. Bit-exact: slot indices, slot tables (feature,
last_use, admit_seq), free counts, error classes; host rows equal the reference's fp64
rows rounded to fp32."""
import numpy as np
import pytest

import paper_2104_08542_b200 as sb
from oracle_lib import ref, ref_available

pytestmark = pytest.mark.gpu

EMPTY = np.iinfo(np.uint64).max


def test_cache_trace_golden(golden):
    tr = golden["cache_trace"]
    c = sb.CacheBuffer(tr["capacity"], tr["dim"], seed=tr["seed"], key_space=64)
    for op in tr["ops"]:
        kind, f, step = op[0], op[1], op[2]
        if kind == "admit":
            assert int(c.admit([f], step)[0]) == op[3], op
        elif kind == "touch":
            c.touch([f], step)
        else:  # the trace clears needed_soon first (admission sets it)
            c.set_needed_soon([f], False)
            c.evict([f])
            assert op[3] == 0
    f, lu, seq, _, _ = c.slots()
    want = [EMPTY if x < 0 else x for x in tr["final_features"]]
    assert f.tolist() == want
    occ = f != EMPTY
    assert lu[occ].tolist() == np.array(tr["final_last_use"])[occ].tolist()
    assert seq[occ].tolist() == np.array(tr["final_admit_seq"])[occ].tolist()
    c.close()


def test_eviction_safety_is_a_logic_error(golden):
    assert golden["eviction_safety"]["needed_soon_status"] == 3
    assert golden["eviction_safety"]["pinned_status"] == 3
    c = sb.CacheBuffer(4, 4, key_space=100)
    c.admit([10, 20], 0)
    with pytest.raises(sb.LogicError, match="lookahead window"):
        c.evict([10])  # admitted => needed_soon (cache_buffer.cpp:44)
    c.set_needed_soon([20], False)
    c.pin([20])
    with pytest.raises(sb.LogicError, match="pinned"):
        c.evict([20])
    with pytest.raises(sb.LogicError, match="non-resident"):
        c.evict([30])
    with pytest.raises(sb.LogicError, match="already resident"):
        c.admit([20], 1)
    c.admit([30, 40], 1)
    with pytest.raises(sb.LogicError, match="no free slot"):
        c.admit([50], 1)
    assert c.occupancy() == {"capacity": 4, "occupied": 4, "free": 0, "pinned": 1,
                             "needed_soon": 3}
    assert c.occupancy_diagnostics() == "capacity=4 occupied=4 free=0 pinned=1 needed_soon=3"
    c.close()


def test_manager_step_paper_example():
    """SPEC.md:195 / PAPER.md:312-318: final cache [7,3,2,5,4,6,12,13,14,15,9,8], 1 evicted."""
    c = sb.CacheBuffer(12, 4, key_space=100)
    c.admit([1, 3, 2, 5, 4, 6, 12, 13, 14, 15, 9], 0)
    c.pin([3, 2, 5, 4])
    out = c.prepare(1, [6, 7, 8], window_ids=[6, 7, 8])
    assert out == {"owned": 3, "hits": 1, "admitted": 2, "evicted": 1, "refilled": 0}
    f = c.slots()[0]
    assert f.tolist() == [7, 3, 2, 5, 4, 6, 12, 13, 14, 15, 9, 8]
    # the evicted feature 1 now lives in the host pool with its initial row
    rows, st = c.peek([1])
    want = sb.initial_embedding(7, 1, 4)
    assert np.array_equal(rows[0, :4], want.astype(np.float32)) and st[0] == 0
    assert not rows[0, 4:].any()
    # capacity shortfall: every resident slot pinned or needed -> RunError, nothing moves
    c.pin([7, 6, 12, 13, 14, 15, 9, 8])
    before = c.slots()[0].copy()
    with pytest.raises(sb.RunError, match="capacity deadlock"):
        c.prepare(2, [50, 51])
    assert np.array_equal(c.slots()[0], before)
    c.close()


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_random_ops_vs_reference_cachebuffer():
    """A seeded random mix of admit / evict / touch / pin / unpin / set_needed_soon, with
    the invalid ones included, on the device and on the reference's own CacheBuffer +
    HostStore: identical return codes, slots, tables, free counts and host rows."""
    R = ref()
    cap, dim, seed = 24, 4, 7
    rc_ = R.ref_cache_create(seed, dim, cap)
    c = sb.CacheBuffer(cap, dim, seed=seed, key_space=128)
    rng = np.random.default_rng(5)
    step = 0
    for _ in range(1500):
        step += int(rng.integers(0, 2))
        f = int(rng.integers(0, 48))
        op = rng.choice(["admit", "admit", "evict", "touch", "pin", "unpin", "ns0", "ns1"])
        if op == "admit":
            want = R.ref_cache_admit(rc_, f, step)
            try:
                got = int(c.admit([f], step)[0])
            except sb.LogicError:
                got = -1
            assert got == (want if want >= 0 else -1), (op, f, want, got)
        elif op == "evict":
            want = R.ref_cache_evict(rc_, f)
            try:
                c.evict([f])
                got = 0
            except sb.LogicError:
                got = 3
            assert got == want, (op, f, want, got)
        else:
            if op == "touch":
                want = R.ref_cache_touch(rc_, f, step)
                call = lambda: c.touch([f], step)  # noqa: E731
            elif op in ("pin", "unpin"):
                want = R.ref_cache_pin(rc_, f, 1 if op == "pin" else 0)
                call = (lambda: c.pin([f])) if op == "pin" else (lambda: c.unpin([f]))
            else:
                want = R.ref_cache_set_needed_soon(rc_, f, 1 if op == "ns1" else 0)
                call = lambda: c.set_needed_soon([f], op == "ns1")  # noqa: E731
            try:
                call()
                got = 0
            except sb.LogicError:
                got = 3
            assert got == want, (op, f, want, got)
        assert c.free_count() == R.ref_cache_free_count(rc_)
    feat = np.zeros(cap, np.uint64)
    lu = np.zeros(cap, np.int64)
    seq = np.zeros(cap, np.uint64)
    R.ref_cache_slots(rc_, feat, lu, seq)
    f2, lu2, seq2, _, _ = c.slots()
    assert np.array_equal(f2, feat)
    occ = feat != EMPTY
    assert np.array_equal(lu2[occ], lu[occ]) and np.array_equal(seq2[occ], seq[occ])
    # host rows (HostStore::peek) of every evicted feature
    for f in range(48):
        row = np.zeros(3 * dim)
        st = np.zeros(1, np.int64)
        import ctypes as C
        if R.ref_cache_host_row(rc_, f, row, st.ctypes.data_as(C.POINTER(C.c_int64))) == 0:
            got, gst = c.peek([f])
            assert np.array_equal(got[0], row.astype(np.float32)) and gst[0] == st[0]
    R.ref_cache_destroy(rc_)
    c.close()
