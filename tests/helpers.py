"""Shared test helpers: seeded inputs and tolerance checks (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle import tgnn_oracle as O

# fp32 device path vs f64 reference: BASELINE north star, 1e-4 relative.
REL_TOL = 1e-4


def random_state(num_nodes, d_mem, t, upto, seed=0, frac=0.8):
    """A NodeMemoryState with random memory/mails whose mail events precede `upto`."""
    rng = np.random.default_rng(seed)
    st = O.MemoryState.init(num_nodes, d_mem)
    st.memory[:] = rng.normal(scale=0.5, size=st.memory.shape)
    st.mail_mem[:] = rng.normal(scale=0.5, size=st.mail_mem.shape)
    has = rng.random(num_nodes) < frac
    ev = rng.integers(0, max(upto, 1), has.sum())
    st.mail_event[has] = ev
    st.mail_t[has] = t[ev]
    st.mail_dt[has] = rng.random(has.sum()) * (t[max(upto - 1, 0)] + 1.0) * 0.1
    st.last_update[has] = st.mail_t[has]
    return st


def rel_close(a, b, tol=REL_TOL, floor=1e-6):
    """max|a-b| <= tol * max(|b|) + floor (per tensor)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    err = np.abs(a - b).max() if a.size else 0.0
    scale = np.abs(b).max() if b.size else 0.0
    return err <= tol * scale + floor, err, scale


def ocfg(mc):
    return mc if isinstance(mc, O.ModelConfig) else O.ModelConfig(**mc.__dict__)


def tensor_slices(mc):
    out, at = {}, 0
    for name, shape in O.tensor_shapes(ocfg(mc)):
        k = int(np.prod(shape))
        out[name] = slice(at, at + k)
        at += k
    return out
