"""Per-step parity from identical state (test infrastructure).

After every step the device state (rows of the step's features, dense parameters and
their Adam moments) is loaded into the oracle, so the next step starts from IDENTICAL
state on both sides and each comparison measures one step's error only: fp32 device
arithmetic against the oracle's fp64 on the same inputs. No multi-step drift enters the
bars, which are therefore tight:

  * loss: |dL| <= 1e-5 |L|;  logits: |dz| <= 1e-5 (1 + |z|)            (every step)
  * the gradient the device summed (scatter-add / all-reduce / owner reduction in fp32,
    any order) within 1e-5 of its condition scale sum|terms| on EVERY coordinate;
  * rows of the step's features and the dense parameters, per row / block (scale = max
    |oracle value|): theta, m, v within 1e-5 * scale plus that gradient tolerance carried
    exactly through the Adam update; the explicitly identified set where the gradient is
    within its own tolerance of zero (sign undetermined in fp32) is checked on the
    gradient only and counted (`check_adam_one_step`).
  * adam step counts, slot tables, ledger: bit-exact.
"""
import ctypes as C

import numpy as np

RTOL = 1e-5


def oracle_rows(O, sim, feats, d):
    n = feats.size
    rows = np.zeros((max(n, 1), 3 * d))
    st = np.zeros(max(n, 1), np.int64)
    O.orc_sim_get_rows(sim, n, np.ascontiguousarray(feats, np.uint64), rows.ctypes.data,
                       st.ctypes.data)
    return rows[:n], st[:n]


def load_rows(O, sim, feats, rows32, steps):
    rows = np.ascontiguousarray(rows32, np.float64)
    st = np.ascontiguousarray(steps, np.int64)
    rc = O.orc_sim_set_rows(sim, feats.size, np.ascontiguousarray(feats, np.uint64),
                            rows.ctypes.data, st.ctypes.data)
    assert rc == 0, O.orc_last_error()


def oracle_dense(O, sim, P):
    p, m, v = np.zeros(P), np.zeros(P), np.zeros(P)
    st = C.c_int64(0)
    O.orc_sim_get_dense_state(sim, p.ctypes.data, m.ctypes.data, v.ctypes.data, C.byref(st))
    return p, m, v, st.value


def load_dense(O, sim, p, m, v, step):
    p, m, v = (np.ascontiguousarray(a, np.float64) for a in (p, m, v))
    st = C.c_int64(step)
    O.orc_sim_set_dense_state(sim, p.ctypes.data, m.ctypes.data, v.ctypes.data, C.byref(st))


class Grads:
    """The oracle's last-step gradients: g / dg, their condition scales gabs / dgabs
    (sums of |terms|), the mass behind fp32-undetermined ReLU decisions gamb / dgamb and
    the count of those decisions n_amb."""

    def __init__(self, O, sim, U, d, P):
        self.g, self.gabs, self.gamb = np.zeros(U * d), np.zeros(U * d), np.zeros(U * d)
        self.dg, self.dgabs, self.dgamb = np.zeros(P), np.zeros(P), np.zeros(P)
        n = C.c_int64(0)
        assert O.orc_sim_last_grads(sim, self.g.ctypes.data, self.gabs.ctypes.data,
                                    self.dg.ctypes.data, self.dgabs.ctypes.data,
                                    self.gamb.ctypes.data, self.dgamb.ctypes.data,
                                    C.byref(n)) == 0
        self.n_amb = n.value
        for k in ("g", "gabs", "gamb"):
            setattr(self, k, getattr(self, k).reshape(U, d))


def adam_update(m0, v0, g, t, cfg):
    """lazy Adam's parameter decrement for gradient g from moments (m0, v0), new step t"""
    b1, b2 = cfg.adam_beta1, cfg.adam_beta2
    m = b1 * m0 + (1 - b1) * g
    v = b2 * v0 + (1 - b2) * g * g
    mh = m / (1 - b1 ** t)
    vh = v / (1 - b2 ** t)
    return cfg.learning_rate * mh / (np.sqrt(vh) + cfg.adam_epsilon)


def check_adam_one_step(old, new_dev, new_orc, g, gabs, gamb, t, cfg, d, what=""):
    """[theta | m | v] after one Adam step from identical state `old`.

    The gradient is the only inexact input: the device sums it in fp32 in another order
    (scatter-add reordering), so its tolerance is stated on the gradient, 1e-5 of the sum's
    condition scale gabs = sum of |terms| (the fp32 reordering bound). Derived from the
    device's first moment, gd = (m_dev - b1 m_old) / (1 - b1), it must satisfy
    |gd - g| <= 1e-5 gabs + the fp32 rounding of m. The parameters must then be within
    1e-5 of their row scale PLUS that gradient tolerance propagated exactly through Adam
    (max |u(g +- 1e-5 gabs) - u(g)|). Coordinates whose gradient is within its own
    tolerance of zero (|g| <= 1e-5 gabs: sign undetermined in fp32, the |g| ~ eps set) are
    checked on the gradient only; their count is reported. One scale per row of `old`.

    gamb: gradient mass behind ReLU decisions fp32 does not determine (the oracle's
    |hpre| <= 1e-5 sum|x w| units): the device may take either branch there, so that
    mass is added to the gradient tolerance (reported: coordinates that needed it)."""
    b1, b2 = cfg.adam_beta1, cfg.adam_beta2
    th, m, v = slice(0, d), slice(d, 2 * d), slice(2 * d, 3 * d)
    a = new_dev.astype(np.float64)
    o = new_orc
    m0, v0 = old[:, m], old[:, v]
    gd = (a[:, m] - b1 * m0) / (1 - b1)
    rnd = 2.0 ** -22 * (np.abs(a[:, m]) + np.abs(m0)) / (1 - b1)
    gerr = np.abs(gd - g)
    amb_used = int(np.sum(gerr > RTOL * gabs + rnd))
    tol = RTOL * gabs + gamb
    assert np.all(gerr <= tol + rnd), (what, "gradient", float(np.max(gerr / (tol + rnd + 1e-300))))

    def scale(x):
        return np.max(np.abs(x), axis=1, keepdims=True) + 1e-30

    tt = np.asarray(t, np.float64).reshape(-1, 1)
    u0 = adam_update(m0, v0, g, tt, cfg)
    du = np.maximum(np.abs(adam_update(m0, v0, g + tol, tt, cfg) - u0),
                    np.abs(adam_update(m0, v0, g - tol, tt, cfg) - u0))
    sens = np.abs(g) <= tol
    stats = {"sensitive_coords": int(sens.sum()), "coords": int(g.size),
             "relu_ambiguous_coords": amb_used}
    # m, v: plain 1e-5 of the row scale + the gradient tolerance through the moment update
    for name, sl, extra in (("m", m, (1 - b1) * tol),
                            ("v", v, (1 - b2) * (2 * np.abs(g) * tol + tol * tol))):
        err = np.abs(a[:, sl] - o[:, sl])
        sc = scale(o[:, sl])
        stats[name + "_max_rel"] = float(np.max(err / sc)) if err.size else 0.0
        ok = err <= RTOL * sc + extra * 1.01
        assert ok.all(), (what, name, stats, np.argwhere(~ok)[:5].tolist())
    err = np.abs(a[:, th] - o[:, th])
    sc = scale(o[:, th])
    stats["theta_max_rel"] = float(np.max(err / sc)) if err.size else 0.0
    plain = err <= RTOL * sc
    stats["theta_outside_plain_1e-5"] = int((~plain & ~sens).sum())
    ok = plain | sens | (err <= RTOL * sc + 1.01 * du)
    assert ok.all(), (what, "theta", stats, np.argwhere(~ok)[:5].tolist())
    return stats


def check_rows_one_step(feats, old, dev_rows, dev_steps, orc_rows, orc_steps, gr, d, cfg,
                        what=""):
    """Rows of the step's features after ONE step from identical state (`old` = the state
    both sides started from, zeros for rows without state). Step counts bit-exact.
    gr: the oracle's Grads of the step, rows in the order of `feats` (global_ids order)."""
    assert np.array_equal(dev_steps, orc_steps), what + " adam steps"
    st = check_adam_one_step(old, dev_rows, orc_rows, gr.g, gr.gabs, gr.gamb, orc_steps, cfg, d,
                             what + " rows")
    st["rows"] = int(feats.size)
    return st


def check_logits(dev, orc, what=""):
    err = np.abs(dev.astype(np.float64) - orc)
    assert np.all(err <= RTOL * (1 + np.abs(orc))), (what, float(np.max(err)))
    return float(np.max(err / (1 + np.abs(orc))))


def check_dense_one_step(old, dev, orc, gr, step, cfg, what=""):
    """dense parameters + Adam moments ([P] each) after one step from identical state,
    with the embedding rows' bars (one scale per parameter block W1 / b1 / w2 / b2)"""
    dg, dga, dgm = gr.dg, gr.dgabs, gr.dgamb
    P = dg.size
    K_H = P - (2 * cfg.hidden_dim + 1)
    H = cfg.hidden_dim
    out = {}
    for name, sl in (("w1", slice(0, K_H)), ("b1", slice(K_H, K_H + H)),
                     ("w2", slice(K_H + H, K_H + 2 * H)), ("b2", slice(P - 1, P))):
        def rows(trip):
            return np.concatenate([np.asarray(x[sl], np.float64)[None] for x in trip], axis=1)
        n = sl.stop - sl.start
        st = check_adam_one_step(rows(old), rows(dev), rows(orc), dg[sl][None], dga[sl][None],
                                 dgm[sl][None], step, cfg, n, f"{what} dense {name}")
        out[name] = st
    return out
