"""Multi-rank runs (i x j x k trainers) against the reference's threaded
run_training on the same stream and seeds.

Two exchange backends, both behind the same C ABI:
  local  every rank a host thread of one process on cuda:0, joined through the
         in-process hub (tgnn_run_local_init; ascending-rank device reductions,
         the reference's own summation order) -- runs on ANY GPU box, so the
         driver's 1-GPU test pass covers every i x j x k shape;
  nccl   one process per GPU under torchrun; generated only for shapes the box
         has enough GPUs for (gpurun --gpus 2/4).
"""
from __future__ import annotations

import json
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


_NGPUS = ngpus()


def backends(T_):
    """local always; nccl when the box has a GPU per rank (collection time)."""
    return ["local"] + (["nccl"] if _NGPUS >= T_ else [])


def launch(script, T_, backend, args, port, timeout=900, env=None):
    if backend == "local":
        cmd = [sys.executable, os.path.join(ROOT, "tests", script), "--backend", "local"] + args
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={T_}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", script),
               "--backend", "nccl"] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]


def shape_params(shapes):
    return [pytest.param(*s, b, id=f"{s[0]}x{s[1]}x{s[2]}-{b}") for s in shapes for b in backends(s[0] * s[1] * s[2])]


SHAPES = [(1, 1, 2, 2), (2, 1, 1, 2), (1, 2, 1, 2), (2, 1, 2, 2), (1, 2, 2, 3), (1, 1, 4, 4), (4, 1, 1, 2),
          (1, 4, 1, 2), (2, 2, 2, 2)]


@pytest.mark.parametrize("i,j,k,epochs,backend", shape_params(SHAPES))
def test_parallel_run_matches_reference(i, j, k, epochs, backend, tmp_path):
    T_ = i * j * k
    out = tmp_path / "r.npz"
    launch("mp_worker.py", T_, backend, ["--i", str(i), "--j", str(j), "--k", str(k), "--epochs", str(epochs),
                                         "--out", str(out)], 29500 + 7 * i + 3 * j + k)
    res = np.load(out)
    assert bool(res["replicas_identical"])  # every rank holds bitwise-identical weights
    rg = ref.RefGraph.synthetic(20, 120, d_e=2, seed=21)
    _, _, t, _ = rg.export(feats=False)
    mc = O.ModelConfig(d_mem=3, d_time=2, d_static=2, d_attn=3, d_hidden=2, d_e=2, n_neighbors=2,
                       num_nodes=20, max_t=float(t[-1]))
    tc = ref.train_cfg(i=i, j=j, k=k, local_batch=15, epochs=epochs, seed=3, lr_base=1e-3)
    rr = rg.run(mc, tc, 0, 90, sequential=False)
    assert int(res["barriers"]) == rr["barriers"]
    # barrier 0 runs on the initial weights: the fp32 step itself within 1e-4
    assert abs(res["losses"][0] - rr["barrier_loss"][0]) <= 1e-4 * abs(rr["barrier_loss"][0])
    # later barriers follow fp32 vs f64 Adam trajectories (dense Adam turns
    # rounding-level gradient differences into lr-sized steps on near-zero
    # gradients, SURVEY 7 hard part 10)
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


_STINT = [s for s in [(1, 2, 1, 2), (2, 2, 1, 2)] if _NGPUS >= s[0] * s[1] * s[2]]
if _STINT:  # the captured stint graphs exist on the NCCL backend only (>= 2 GPUs)
    @pytest.mark.parametrize("i,j,k,epochs", _STINT)
    def test_stint_graphs_bitwise_equal_direct(i, j, k, epochs, tmp_path):
        """j > 1 over NCCL: the per-position stint graphs reproduce the direct path bitwise."""
        T_ = i * j * k
        res = {}
        for mode in ("graph", "direct"):
            out = tmp_path / f"{mode}.npz"
            launch("mp_worker.py", T_, "nccl", ["--i", str(i), "--j", str(j), "--k", str(k), "--epochs", str(epochs),
                                                "--out", str(out)] + (["--direct"] if mode == "direct" else []),
                   29600 + 7 * i + 3 * j + k + (mode == "direct"))
            res[mode] = np.load(out)
        for key in ("losses", "params", "oplog"):
            assert np.array_equal(res["graph"][key], res["direct"][key]), key


if _NGPUS >= 2:  # the NCCL graph pipeline at C2 dimensions (one process per GPU)
    @pytest.mark.parametrize("i,j,k", [(1, 1, 2), (2, 1, 1)])
    def test_graph_pipeline_bitwise_equal_direct_at_c2_dims(i, j, k, tmp_path):
        """k = 2 / i = 2 at Reddit dimensions over 40 barriers: the production
        multi-barrier graphs (deferred tail update, head bucket on its own
        communicator, i-axis exchange on its own stream) reproduce the direct
        path bitwise and every replica stays identical."""
        T_ = i * j * k
        res = {}
        for mode in ("graph", "direct"):
            out = tmp_path / f"{mode}.npz"
            launch("mp_worker.py", T_, "nccl", ["--i", str(i), "--j", str(j), "--k", str(k), "--epochs", str(T_),
                                                "--shape", "reddit", "--local-batch", "600", "--train-end", "24000",
                                                "--out", str(out)] + (["--direct"] if mode == "direct" else []),
                   29800 + 7 * i + k + (mode == "direct"))
            res[mode] = np.load(out)
            assert bool(res[mode]["replicas_identical"])
        for key in ("losses", "params"):
            assert np.array_equal(res["graph"][key], res["direct"][key]), key


# acceptance criterion 8 (ref/tests/acceptance.cpp:435-458): final val
# MRR at 525,000 traversed events. The reference's anchors (0.8767 / 0.8824 /
# 0.8368 at training seed 5, tolerances 0.02 / 0.02 / 0.05) are single samples of
# a chaotic 150-epoch trajectory: the unmodified reference itself moves by up to
# 0.03 between training seeds (tests/golden/convergence_ref.json, made by
# oracle/_ref), and an fp32 run follows a different trajectory from seed 5 on.
# So the device is held to the reference's tolerance on the MEAN over the same
# eight training seeds, and every seed to at least the reference's worst seed
# less three tolerances (per-seed pairs differ by up to ~0.06 either way).
CONV_SEEDS = list(range(5, 13))
CONV_TOL = {(1, 1, 1): 0.02, (1, 1, 4): 0.02, (1, 4, 1): 0.05}


def conv_reference(i, j, k):
    with open(os.path.join(ROOT, "tests", "golden", "convergence_ref.json")) as f:
        row = json.load(f)[f"{i}x{j}x{k}"]
    return np.array([row[str(sd)] for sd in CONV_SEEDS])


@pytest.mark.parametrize("i,j,k,backend", [pytest.param(1, 1, 1, "local", id="1x1x1-local")] +
                         shape_params([(1, 1, 4), (1, 4, 1)]))
def test_convergence_matches_reference_anchors(i, j, k, backend, tmp_path):
    T_ = i * j * k
    out = tmp_path / "c.npz"
    launch("mp_convergence.py", T_, backend, ["--i", str(i), "--j", str(j), "--k", str(k), "--out", str(out),
                                             "--seeds", ",".join(map(str, CONV_SEEDS))],
           29700 + 7 * i + 3 * j + k, timeout=1500)
    res = np.load(out)
    assert np.all(res["traversed"] == 525000)
    want = conv_reference(i, j, k)
    tol = CONV_TOL[(i, j, k)]
    got = res["mrr"]
    print(f"\n({i},{j},{k}) [{backend}] device MRR per seed {np.round(got, 4).tolist()} mean {got.mean():.4f}; "
          f"reference {want.tolist()} mean {want.mean():.4f}")
    assert abs(got.mean() - want.mean()) <= tol
    assert np.all(got >= want.min() - 3 * tol)


# acceptance criterion 4 (ref/tests/acceptance.cpp:265-328): small_graph_500(41, 1),
# model_for(g, 6, 3, 2, 6, 3), k = 4, batch 25, 4 epochs, seed 9, frozen weights
SNAP_GRAPH = dict(nodes=120, events=500, d_e=1, seed=41)
SNAP_MODEL = dict(d_mem=6, d_time=3, d_static=2, d_attn=6, d_hidden=6, d_e=1, n_neighbors=3, num_nodes=120)


def snapshot_reference():
    """The reference run_training's snapshots (copy, sweep, segment, memory, last_update)."""
    rg = ref.RefGraph.synthetic(SNAP_GRAPH["nodes"], SNAP_GRAPH["events"], d_e=SNAP_GRAPH["d_e"],
                                seed=SNAP_GRAPH["seed"])
    _, _, t, _ = rg.export(feats=False)
    mc = O.ModelConfig(max_t=float(t[-1]), **SNAP_MODEL)
    tc = ref.train_cfg(k=4, local_batch=25, epochs=4, seed=9, lr_base=0.0)
    return rg, mc, ref.run_snapshots(rg, mc, tc, 0, 400)


def test_segment_snapshots_match_reference(tmp_path):
    """Acceptance criterion 4 on the in-process backend (4 ranks on cuda:0):
    k = 4 memory copies, frozen weights (lr_base = 0), segment snapshots
    (DaemonOp::Snapshot, memory_daemon.hpp:94-105). Every snapshot of every
    copy matches the reference run_training's (same sweep/segment list, memory
    within 1e-4 normwise and elementwise, last_update exactly); the reference
    snapshots themselves are pinned to their fresh-replay oracle in
    tests/test_oracle_golden.py::test_reference_snapshots_equal_fresh_replay."""
    out = tmp_path / "s.npz"
    code = f"""
import sys, numpy as np
sys.path.insert(0, {ROOT!r})
import paper_2307_07649_b200 as T
s = T.gen_synthetic(T.SynthParams(**{SNAP_GRAPH!r}))
def body(rank, hub):
    ctx = T.Context(0)
    g = T.TemporalGraph.from_stream(ctx, s)
    mc = T.ModelConfig(max_t=float(s.t[-1]), **{SNAP_MODEL!r})
    tc = T.TrainConfig(k=4, local_batch=25, epochs=4, seed=9, lr_base=0.0)
    run = T.Run(ctx, g, mc, tc, 0, 400, rank=rank, nranks=4, segment_snapshots=True)
    run.local_init(hub)
    run.step(run.barriers)
    sn = run.snapshots()
    run.close(); g.close(); ctx.close()
    return sn
res = T.run_ranks(body, 4)
np.savez({str(out)!r}, **{{f"{{k}}_{{r}}": v for r, sn in enumerate(res) for k, v in sn.items()}})
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = np.load(out)
    _, _, (meta, mem, lu) = snapshot_reference()
    assert len(meta) == 16  # acceptance.cpp criterion 4 reports 16 snapshots
    compared = 0
    for grp in range(4):  # rank == memory copy at (1, 1, 4)
        sel = meta[:, 0] == grp
        assert np.array_equal(res[f"meta_{grp}"], meta[sel][:, 1:]), grp
        for x, (w_mem, w_lu) in enumerate(zip(mem[sel], lu[sel])):
            o_mem, o_lu = res[f"memory_{grp}"][x], res[f"last_update_{grp}"][x]
            assert np.array_equal(o_lu, w_lu), (grp, x)
            err = np.abs(o_mem - w_mem)
            scale = np.abs(w_mem).max()
            assert err.max() <= 1e-4 * scale + 1e-7, (grp, x, err.max(), scale)
            # elementwise: 1e-4 relative to each element, floored at a tenth of
            # the tensor's largest magnitude (the GRU replay compounds fp32
            # rounding over up to 16 batches)
            assert np.all(err <= 1e-4 * np.maximum(np.abs(w_mem), 0.1 * scale)), (grp, x, err.max())
            compared += 1
    assert compared == 16
