"""Runs a few deterministic steps on cuda:0 and saves the final state (tests/test_gpu_parity.py
test_launch_switches_are_bit_identical launches it under different launch / scheduling
switches, which are read once per process)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main(out, mode):
    import paper_2104_08542_b200 as sb
    cfg = sb.Config(num_workers=1, batch_size_per_worker=1024, num_fields=12, embedding_dim=16,
                    vocabulary_size=100_000, cache_capacity=100_000, hidden_dim=32,
                    zipf_exponent=1.05)
    cfg.apply("deterministic", "1")
    cfg.apply("mode", mode)
    gen = sb.SyntheticGenerator(cfg)
    tr = sb.Trainer(cfg)
    losses = [tr.step(t, *gen.generate(t)) for t in range(6)]
    f, r, s = tr.snapshot()
    p, m, v, ds = tr.dense_state()
    np.savez(out, losses=np.array(losses), f=f, r=r, s=s, p=p, m=m, v=v)
    tr.close()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
