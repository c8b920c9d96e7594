"""Criteo TSV ingest (CriteoReader, core/src/criteo.cpp:25-98).

CPU part: the oracle's C restatement (oracle/sfctr_oracle.c) against the reference's
own compiled CriteoReader (oracle/_ref) on generated TSV files with the reader's edge
cases — hashed ids, labels, wrap-around batches, DataError line numbers and messages —
all BIT-EXACT. GPU part: the device parser through the C-ABI against the oracle, same
bar, including multi-chunk streaming (lines cut at chunk boundaries)."""
import os

import numpy as np
import pytest

import paper_2104_08542_b200 as sb
from oracle_lib import (make_criteo_tsv, oracle, oracle_criteo, ref, ref_available)

needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


def _ref_read(path, vocab, workers, batch, steps):
    import ctypes as C
    R = ref()
    rc = C.c_int(0)
    h = R.ref_criteo_open(str(path).encode(), 26, vocab, workers, batch, C.byref(rc))
    if not h:
        return rc.value, R.ref_last_error().decode(), None
    rows = R.ref_criteo_rows(h)
    out = []
    G = workers * batch
    for s in range(steps):
        f = np.zeros(G * 26, np.uint64)
        y = np.zeros(G, np.uint8)
        R.ref_criteo_read_batch(h, s, f, y)
        out.append((f, y))
    R.ref_criteo_destroy(h)
    return 0, rows, out


def _orc_batches(data, vocab, G, steps):
    f, y = oracle_criteo(data, vocab)
    rows = len(y)
    O = oracle()
    out = []
    for s in range(steps):
        of = np.zeros(G * 26, np.uint64)
        ol = np.zeros(G, np.uint8)
        O.orc_criteo_read_batch(f, y, rows, s, G, of, ol)
        out.append((of, ol))
    return rows, out


def test_token_hash_golden():
    # survey golden: fnv1a64("68fd1e64") = 0x1ae7327a0f5691dd (mod 1e6 = 18461)
    assert oracle().orc_fnv1a64(b"68fd1e64", 8) == 0x1AE7327A0F5691DD
    assert sb.CriteoReader.token_hash("68fd1e64") == 0x1AE7327A0F5691DD
    assert 0x1AE7327A0F5691DD % 1_000_000 == 18461


@needs_ref
@pytest.mark.parametrize("seed,rows,vocab", [(0, 50, 1000), (1, 333, 1_000_000), (2, 1, 97),
                                             (3, 2000, 33_800_000)])
def test_oracle_matches_reference_reader(tmp_path, seed, rows, vocab):
    data = make_criteo_tsv(rows, seed)
    p = tmp_path / "day.tsv"
    p.write_bytes(data)
    W, b, steps = 2, 7, 5
    rc, nrows, ref_b = _ref_read(p, vocab, W, b, steps)
    assert rc == 0, nrows
    orows, orc_b = _orc_batches(data, vocab, W * b, steps)
    assert orows == nrows
    for (rf, ry), (of, oy) in zip(ref_b, orc_b):
        assert np.array_equal(rf, of) and np.array_equal(ry, oy)
    assert ref().ref_criteo_token_hash(b"68fd1e64", 8) == 0x1AE7327A0F5691DD


BAD_CASES = [
    # (mutation, expected message tail)
    (lambda ls: ls.__setitem__(3, ls[3] + "\textra"), "expected 40 tab-separated columns, got 41"),
    (lambda ls: ls.__setitem__(5, "\t".join(ls[5].split("\t")[:20])),
     "expected 40 tab-separated columns, got 20"),
    (lambda ls: ls.__setitem__(2, "2" + ls[2][1:]), "label must be 0 or 1, got '2'"),
    (lambda ls: ls.__setitem__(4, "10" + ls[4][1:]), "label must be 0 or 1, got '10'"),
    (lambda ls: ls.__setitem__(6, "\t" + ls[6][2:]), "label must be 0 or 1, got ''"),
]


def _bad_file(i):
    lines = make_criteo_tsv(12, 100 + i, edge_cases=False).decode().split("\n")
    BAD_CASES[i][0](lines)
    return "\n".join(lines).encode()


@needs_ref
@pytest.mark.parametrize("i", range(len(BAD_CASES)))
def test_oracle_errors_match_reference(tmp_path, i):
    data = _bad_file(i)
    p = tmp_path / "bad.tsv"
    p.write_bytes(data)
    rc, msg, _ = _ref_read(p, 1000, 1, 4, 1)
    assert rc == 2  # DataError
    with pytest.raises(ValueError) as e:
        oracle_criteo(data, 1000)
    line, tail = e.value.args
    assert msg == f"{p}:{line}: {tail}"
    assert tail == BAD_CASES[i][1]


@needs_ref
def test_no_data_rows(tmp_path):
    p = tmp_path / "empty.tsv"
    p.write_bytes(b"\n\r\n\n")
    rc, msg, _ = _ref_read(p, 1000, 1, 4, 1)
    assert rc == 2 and msg == f"{p}: no data rows"
    with pytest.raises(ValueError):
        oracle_criteo(b"\n\r\n\n", 1000)


# ---------------- device ----------------

def _cfg(vocab, W=2, b=7, fields=26):
    return sb.Config(num_workers=W, batch_size_per_worker=b, num_fields=fields,
                     vocabulary_size=vocab)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,rows,vocab,chunk", [(0, 50, 1000, None), (1, 3000, 1_000_000, None),
                                                   (2, 3000, 33_800_000, 8192),
                                                   (3, 20000, 1 << 31, 65536)])
def test_device_parse_matches_oracle(tmp_path, monkeypatch, seed, rows, vocab, chunk):
    if chunk:
        monkeypatch.setenv("SFCTR_CRITEO_CHUNK", str(chunk))
    data = make_criteo_tsv(rows, seed)
    p = tmp_path / "day.tsv"
    p.write_bytes(data)
    W, b, steps = 2, 7, 6
    rd = sb.CriteoReader(p, _cfg(vocab, W, b))
    orows, orc_b = _orc_batches(data, vocab, W * b, steps)
    assert rd.row_count() == orows
    for s in range(steps):
        f, y = rd.read_batch(s)
        assert np.array_equal(f, orc_b[s][0]) and np.array_equal(y, orc_b[s][1]), s
        f1, y1 = rd.read_batch(s, row0=b, nrows=b)  # rank 1's rows
        assert np.array_equal(f1, orc_b[s][0][b * 26:]) and np.array_equal(y1, orc_b[s][1][b:])
    # the whole table: one batch spanning every row
    big = sb.CriteoReader.from_bytes(data, _cfg(vocab, 1, orows))
    f, y = big.read_batch(0)
    of, oy = oracle_criteo(data, vocab)
    assert np.array_equal(f, of) and np.array_equal(y, oy)
    st = big.stats()
    assert st["bytes"] >= len(data) and st["lines"] >= orows


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(BAD_CASES)))
@pytest.mark.parametrize("chunk", [None, 4096])
def test_device_errors_match_oracle(tmp_path, monkeypatch, i, chunk):
    if chunk:
        monkeypatch.setenv("SFCTR_CRITEO_CHUNK", str(chunk))
    data = _bad_file(i)
    p = tmp_path / "bad.tsv"
    p.write_bytes(data)
    with pytest.raises(ValueError) as e:
        oracle_criteo(data, 1000)
    line, tail = e.value.args
    with pytest.raises(sb.DataError) as d:
        sb.CriteoReader(p, _cfg(1000))
    assert str(d.value) == f"{p}:{line}: {tail}"


@pytest.mark.gpu
def test_device_config_errors(tmp_path):
    with pytest.raises(sb.ConfigError):
        sb.CriteoReader(tmp_path / "missing.tsv", _cfg(1000))
    p = tmp_path / "x.tsv"
    p.write_bytes(make_criteo_tsv(3, 0))
    with pytest.raises(sb.ConfigError):
        sb.CriteoReader(p, _cfg(1000, fields=39))
    with pytest.raises(sb.DataError):
        sb.CriteoReader.from_bytes(b"\n\n", _cfg(1000), name="e")


def test_device_entry_points_exported():
    lib = sb.sfctr.lib()
    for n in ("sfctr_criteo_open", "sfctr_criteo_open_buffer", "sfctr_criteo_read_batch",
              "sfctr_criteo_read_batch_device", "sfctr_criteo_row_count", "sfctr_criteo_stats",
              "sfctr_criteo_token_hash", "sfctr_criteo_destroy"):
        assert hasattr(lib, n)
    assert os.path.exists(os.path.join(os.path.dirname(sb.__file__), "libsfctr_b200.so"))


@pytest.mark.gpu
def test_batch_source_data_key(tmp_path):
    """config key data=criteo:<path> feeds the trainer through the batch source (the
    reference's pipeline data loader); data=synthetic is the generator, bit for bit."""
    data = make_criteo_tsv(3000, seed=4)
    p = tmp_path / "day.tsv"
    p.write_bytes(data)
    cfg = sb.Config(num_workers=2, batch_size_per_worker=256, num_fields=26, embedding_dim=8,
                    vocabulary_size=50000, cache_capacity=20000, hidden_dim=16)
    cfg.apply("data", f"criteo:{p}")
    src = sb.BatchSource(cfg)
    rd = sb.CriteoReader(str(p), cfg)
    for step in (0, 5, 11):
        f1, y1 = src.read(step)
        f2, y2 = rd.read_batch(step)
        assert np.array_equal(f1, f2) and np.array_equal(y1, y2)
    tr = sb.Trainer(cfg)
    for step in range(3):
        loss = tr.step(step, *src.read(step))
        assert np.isfinite(loss)
    tr.close()
    src.close()
    cfg.apply("data", "synthetic")
    src = sb.BatchSource(cfg)
    gen = sb.SyntheticGenerator(cfg)
    f1, y1 = src.read(3, 256, 256)
    f2, y2 = gen.generate(3, 256, 256)
    assert np.array_equal(f1, f2) and np.array_equal(y1, y2)
    src.close()
