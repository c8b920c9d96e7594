"""CPU tests of the C-ABI library (no GPU needed): it loads, exports every
symbol include/sfctr_b200.h declares, keeps the reference's config grammar,
defaults and error classes, and fails loudly (CudaError) instead of falling
back when no device is present."""
import os
import re

import numpy as np
import pytest

import paper_2104_08542_b200 as sb
from paper_2104_08542_b200 import sfctr
from oracle_lib import ref, ref_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sfctr_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sfctr_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = sfctr.lib()
    syms = declared_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(L, s), s
    bound = {name for name, _, _ in sfctr.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound


def test_abi_version():
    assert sfctr.lib().sfctr_abi_version() == 2


def test_config_defaults_match_reference():
    c = sb.Config()  # config.hpp:44-71
    assert (c.num_workers, c.embedding_dim, c.num_fields, c.batch_size_per_worker) == (4, 16, 26, 256)
    assert (c.vocabulary_size, c.cache_capacity, c.lookahead_depth, c.seed) == (100000, 8192, 1, 7)
    assert (c.learning_rate, c.adam_beta1, c.adam_beta2, c.adam_epsilon) == (1e-3, 0.9, 0.999, 1e-8)
    assert (c.zipf_exponent, c.hidden_dim) == (1.2, 64)
    c.validate()


def test_config_grammar_and_errors(golden, tmp_path):
    # the same statuses the reference's apply_config_entry/validate give (golden config_checks)
    for key, value, status in golden["config_checks"]:
        c = sb.Config()
        try:
            c.apply(key, value)
            c.validate()
            got = 0
        except sb.ConfigError:
            got = 1
        assert got == status, (key, value)
    p = tmp_path / "run.cfg"
    p.write_text("# comment\nworkers = 8\n dim=80 # trailing\n\nvocab=33800000\nsync=alltoall\n")
    c = sb.Config().load(str(p))
    assert c.num_workers == 8 and c.embedding_dim == 80 and c.vocabulary_size == 33800000
    assert c.sync_mode == 1
    p.write_text("workers 8\n")
    with pytest.raises(sb.ConfigError):
        sb.Config().load(str(p))
    with pytest.raises(sb.ConfigError):
        sb.Config().load(str(tmp_path / "missing.cfg"))


def test_core_helpers(golden):
    for s, h in golden["fnv1a64"].items():
        assert format(sb.fnv1a64(s.encode()), "016x") == h
    for base, label, idx, h in golden["derive_seed"]:
        assert format(sb.derive_seed(base, label, idx), "016x") == h
    for p, w, want in golden["allreduce_bytes"]:
        assert sb.allreduce_bytes(p, w) == want
    with pytest.raises(sb.LogicError):
        sb.allreduce_bytes(10, 0)


@pytest.mark.skipif(sb.device_count() > 0, reason="checks the no-GPU behaviour")
def test_no_silent_cpu_fallback():
    cfg = sb.Config(num_workers=1, batch_size_per_worker=4)
    with pytest.raises(sb.CudaError):
        sb.Trainer(cfg)
    with pytest.raises(sb.CudaError):
        sb.virtual_sparse_id(np.arange(4, dtype=np.uint64), 2, 2)
    with pytest.raises(sb.CudaError):
        sb.SyntheticGenerator(cfg)
    with pytest.raises(sb.CudaError):
        sb.initial_embedding(7, 0, 4)


def test_data_source_config_key():
    """config key `data` (config.cpp:146-154) and its validation (config.cpp:74-77), with the
    reference's messages; `deterministic` is a B200 key."""
    c = sb.Config()
    c.apply("data", "criteo:/data/day_0.tsv")
    assert c.data_source == 1 and c.criteo_path == b"/data/day_0.tsv"
    c.validate()
    c.apply("fields", "25")
    with pytest.raises(sb.ConfigError, match="criteo format has 26 categorical fields; set fields=26"):
        c.validate()
    c.apply("data", "synthetic")
    assert c.data_source == 0 and c.criteo_path == b""
    c.validate()
    with pytest.raises(sb.ConfigError, match="expected 'synthetic' or 'criteo:<path>'"):
        sb.Config().apply("data", "parquet:/x")
    c = sb.Config()
    c.apply("data", "criteo:")
    with pytest.raises(sb.ConfigError, match="criteo data source needs a file path"):
        c.validate()
    c = sb.Config()
    c.apply("deterministic", "1")
    assert c.deterministic == 1
    with pytest.raises(sb.ConfigError):
        c.apply("deterministic", "maybe")


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")
def test_data_source_messages_match_reference():
    R = ref()
    for key, value in (("data", "parquet:/x"), ("data", "criteo:")):
        assert R.ref_config_check(key.encode(), value.encode(), 1) == 1
        want = R.ref_last_error().decode()
        c = sb.Config()
        with pytest.raises(sb.ConfigError) as e:
            c.apply(key, value)
            c.validate()
        assert str(e.value) == want, (str(e.value), want)
