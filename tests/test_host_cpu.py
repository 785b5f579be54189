"""CPU: the product library loads, exports every symbol include/tgnn_b200.h
declares, and its host-side restatements (generator, init_params, the i x j x k
schedule) are bit-identical to the reference golden vectors. No GPU needed."""
from __future__ import annotations

import os
import re

import numpy as np
import pytest

import paper_2307_07649_b200 as T
from paper_2307_07649_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = np.load(os.path.join(ROOT, "tests", "golden", "small.npz"))
MODEL = dict(d_mem=6, d_time=4, d_static=3, d_attn=5, d_hidden=4, n_neighbors=5)


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tgnn_b200.h")).read()
    return sorted(set(re.findall(r"\b(tgnn_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    import ctypes
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 40
    for s in syms:
        assert hasattr(lib, s), s
    # and the ctypes table binds exactly the declared surface
    assert set(_lib.SIGNATURES) == set(syms)


def test_generator_bit_identical():
    s = T.gen_synthetic(T.SynthParams(nodes=60, events=800, d_e=4, seed=3))
    assert s.boundary == int(GOLD["boundary"])
    assert np.array_equal(s.src, GOLD["src"]) and np.array_equal(s.dst, GOLD["dst"])
    assert np.array_equal(s.t, GOLD["t"])
    assert np.array_equal(s.efeat, GOLD["efeat"].astype(np.float32))
    s2 = T.gen_synthetic(T.SynthParams(nodes=40, events=300, d_e=2, seed=9, bipartite=False))
    assert s2.boundary == -1
    assert np.array_equal(s2.src, GOLD["nb_src"]) and np.array_equal(s2.dst, GOLD["nb_dst"])
    assert np.array_equal(s2.t, GOLD["nb_t"])


def test_init_params_bit_identical():
    mc = T.ModelConfig(d_e=4, num_nodes=int(GOLD["num_nodes"]), max_t=float(GOLD["t"][-1]), **MODEL)
    p = T.init_params(mc, 7)
    assert p.shape == GOLD["init_params_seed7"].shape
    assert np.array_equal(p, GOLD["init_params_seed7"])
    assert T.param_count(mc) == len(p)


@pytest.mark.parametrize("x", range(7))
def test_schedule_matches_reference(x):
    i, j, k, ep = (int(v) for v in GOLD["sched_shapes"][x])
    tc = T.TrainConfig(i=i, j=j, k=k, local_batch=50, epochs=ep, seed=5)
    act = GOLD[f"sched{x}_active"]
    for r in range(i * j * k):
        nb, q = T.schedule_query(tc, 0, 1234, r)
        assert nb == act.shape[1]
        m = act[r] == 1
        assert np.array_equal(q["active"], act[r])
        for key in ("sub", "slice_begin", "slice_end", "neg_group"):
            assert np.array_equal(q[key][m], GOLD[f"sched{x}_{key}"][r][m]), key
        assert np.array_equal(q["active_trainers"], GOLD[f"sched{x}_active_trainers"])
        assert np.array_equal(q["traversed_after"], GOLD[f"sched{x}_traversed_after"])


def test_schedule_slices_partition_global_batches():
    tc = T.TrainConfig(i=4, j=2, k=1, local_batch=37, epochs=2, seed=1)
    nb, tabs = None, []
    for r in range(8):
        nb, q = T.schedule_query(tc, 100, 2000, r)
        tabs.append(q)
    for b in range(nb):
        for team in range(2):
            rs = [team * 4 + m for m in range(4)]
            if not tabs[rs[0]]["active"][b]:
                continue
            cuts = [(tabs[r]["slice_begin"][b], tabs[r]["slice_end"][b]) for r in rs]
            assert cuts[0][0] == tabs[rs[0]]["batch_begin"][b]
            assert cuts[-1][1] == tabs[rs[0]]["batch_end"][b]
            for a, c in zip(cuts, cuts[1:]):
                assert a[1] == c[0]


def test_config_errors_map_to_exceptions():
    with pytest.raises(T.ConfigError):
        T.schedule_query(T.TrainConfig(i=2, j=1, k=1, p=1, q=1), 0, 100, 0)  # i*j*k != p*q
    with pytest.raises(T.ConfigError):
        T.schedule_query(T.TrainConfig(local_batch=0), 0, 100, 0)
    with pytest.raises(T.ConfigError):
        T.gen_synthetic(T.SynthParams(nodes=1, events=10))


def test_no_silent_cpu_fallback():
    """Without a GPU, device entry points fail loudly (CudaError), never fall back."""
    n = np.zeros(1, np.int32)
    import ctypes
    rc = _lib.lib().tgnn_device_count(ctypes.cast(n.ctypes.data, ctypes.POINTER(ctypes.c_int)))
    assert rc == 0
    if n[0] == 0:
        with pytest.raises(T.CudaError):
            T.Context(0)


def test_checkpoint_byte_compatible(tmp_path):
    """model.ckpt (ref model.hpp:168-222): our writer reproduces the reference's
    bytes, our reader loads the reference's file, and mismatches are refused."""
    mc = T.ModelConfig(d_e=4, num_nodes=int(GOLD["num_nodes"]), max_t=float(GOLD["t"][-1]), **MODEL)
    gold_path = os.path.join(ROOT, "tests", "golden", "small.ckpt")
    out = tmp_path / "model.ckpt"
    T.save_checkpoint(mc, GOLD["run_params"], out)
    assert out.read_bytes() == open(gold_path, "rb").read()
    assert np.array_equal(T.load_checkpoint(mc, gold_path), GOLD["run_params"])
    other = T.ModelConfig(d_e=4, num_nodes=int(GOLD["num_nodes"]), max_t=1.0,
                          **dict(MODEL, d_attn=6))
    with pytest.raises(T.ConfigError, match="manifest mismatch"):
        T.load_checkpoint(other, gold_path)
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(b"not a checkpoint\n")
    with pytest.raises(T.ConfigError, match="bad magic"):
        T.load_checkpoint(mc, bad)
    trunc = tmp_path / "trunc.ckpt"
    trunc.write_bytes(open(gold_path, "rb").read()[:-8])
    with pytest.raises(T.ConfigError, match="truncated payload"):
        T.load_checkpoint(mc, trunc)
    with pytest.raises(T.ConfigError, match="cannot open"):
        T.load_checkpoint(mc, tmp_path / "missing.ckpt")
