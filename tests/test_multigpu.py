"""Multi-GPU (one rank per trainer over NCCL): i x j x k runs against the
reference's threaded run_training on the same stream and seeds. Needs >= 2
GPUs (gpurun --gpus 2/4); skipped otherwise."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import ref
from oracle import tgnn_oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


SHAPES = [(1, 1, 2, 2), (2, 1, 1, 2), (1, 2, 1, 2), (2, 1, 2, 2), (1, 2, 2, 3), (1, 1, 4, 4)]


@pytest.mark.parametrize("i,j,k,epochs", SHAPES)
def test_parallel_run_matches_reference(i, j, k, epochs, tmp_path):
    T_ = i * j * k
    if ngpus() < T_:
        pytest.skip(f"needs {T_} GPUs")
    out = tmp_path / "r.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={T_}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + 7 * i + 3 * j + k),
           os.path.join(ROOT, "tests", "mp_worker.py"), "--i", str(i), "--j", str(j), "--k", str(k),
           "--epochs", str(epochs), "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = np.load(out)
    assert bool(res["replicas_identical"])  # every rank holds bitwise-identical weights
    rg = ref.RefGraph.synthetic(20, 120, d_e=2, seed=21)
    _, _, t, _ = rg.export(feats=False)
    mc = O.ModelConfig(d_mem=3, d_time=2, d_static=2, d_attn=3, d_hidden=2, d_e=2, n_neighbors=2,
                       num_nodes=20, max_t=float(t[-1]))
    tc = ref.train_cfg(i=i, j=j, k=k, local_batch=15, epochs=epochs, seed=3, lr_base=1e-3)
    rr = rg.run(mc, tc, 0, 90, sequential=False)
    assert int(res["barriers"]) == rr["barriers"]
    assert np.abs(res["losses"] - rr["barrier_loss"]).max() <= 1e-3 * np.abs(rr["barrier_loss"]).max()
    lr = 1e-3 * T_
    assert np.abs(res["params"] - rr["params"]).max() <= 2.5 * lr * rr["barriers"]
    assert np.median(np.abs(res["params"] - rr["params"])) <= 1e-5
    # the daemon op-log of every memory copy, byte for byte (memory_daemon.hpp:73,90)
    import paper_2307_07649_b200 as T
    rg.run_oplog(mc, tc, 0, 90, str(tmp_path / "ref"))
    rows = res["oplog"]
    for grp in range(k):
        ours = tmp_path / f"ours.{grp}.oplog"
        T.write_oplog(ours, rows[rows[:, 0] == grp][:, 1:])
        want = (tmp_path / f"ref.{grp}.oplog").read_text()
        assert ours.read_text() == want, grp
        assert ref.validate_oplog(str(ours), i, j)[0]


@pytest.mark.parametrize("i,j,k,epochs", [(1, 2, 1, 2), (2, 2, 1, 2)])
def test_stint_graphs_bitwise_equal_direct(i, j, k, epochs, tmp_path):
    """j > 1: the per-position stint graphs reproduce the direct path bitwise."""
    T_ = i * j * k
    if ngpus() < T_:
        pytest.skip(f"needs {T_} GPUs")
    res = {}
    for mode in ("graph", "direct"):
        out = tmp_path / f"{mode}.npz"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={T_}",
               "--master-addr", "127.0.0.1", "--master-port", str(29600 + 7 * i + 3 * j + k + (mode == "direct")),
               os.path.join(ROOT, "tests", "mp_worker.py"), "--i", str(i), "--j", str(j), "--k", str(k),
               "--epochs", str(epochs), "--out", str(out)] + (["--direct"] if mode == "direct" else [])
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        res[mode] = np.load(out)
    for key in ("losses", "params", "oplog"):
        assert np.array_equal(res["graph"][key], res["direct"][key]), key


# acceptance criterion 8 (ref/tests/acceptance.cpp:435-458): final val
# MRR at 525,000 traversed events; reference anchors and tolerances
ANCHORS = {(1, 1, 1): (0.8767, 0.02), (1, 1, 4): (0.8824, 0.02), (1, 4, 1): (0.8368, 0.05)}


@pytest.mark.parametrize("i,j,k", [(1, 1, 4), (1, 4, 1)])
def test_convergence_matches_reference_anchors(i, j, k, tmp_path):
    T_ = i * j * k
    if ngpus() < T_:
        pytest.skip(f"needs {T_} GPUs")
    out = tmp_path / "c.npz"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={T_}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + 7 * i + 3 * j + k),
           os.path.join(ROOT, "tests", "mp_convergence.py"), "--i", str(i), "--j", str(j), "--k", str(k),
           "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = np.load(out)
    assert int(res["traversed"]) == 525000
    want, tol = ANCHORS[(i, j, k)]
    print(f"\n({i},{j},{k}) device MRR {float(res['mrr']):.4f} vs reference {want}")
    assert abs(float(res["mrr"]) - want) <= tol


def test_peer_allreduce_matches_nccl(tmp_path):
    """TGNN_ALLREDUCE=peer (NVLink peer-memory all-reduce, peer.cu): the same
    run as NCCL up to the summation order -- losses within 1e-6, replicas
    bitwise identical, op-log identical."""
    if ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    res = {}
    for mode in ("peer", "nccl"):
        out = tmp_path / f"{mode}.npz"
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
               "--master-addr", "127.0.0.1", "--master-port", str(29650 + (mode == "nccl")),
               os.path.join(ROOT, "tests", "mp_worker.py"), "--k", "2", "--epochs", "2", "--out", str(out)]
        env = dict(os.environ, TGNN_ALLREDUCE=mode)
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        res[mode] = np.load(out)
        assert bool(res[mode]["replicas_identical"])
    assert np.abs(res["peer"]["losses"] - res["nccl"]["losses"]).max() <= 1e-6
    assert np.array_equal(res["peer"]["oplog"], res["nccl"]["oplog"])
