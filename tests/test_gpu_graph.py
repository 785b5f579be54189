"""GPU: the pipelined CUDA-graph barrier (plan-ahead on an aux stream, edge
projection / root writes / loss / split-K reductions on branch streams,
programmatic dependent launch, fused Adam + weight pack) must be a pure
schedule change: bitwise the same losses and weights as the direct,
single-stream path. A race between branches shows up here first."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2307_07649_b200 as T

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cfg", [dict(nodes=10984, events=60000, d_e=172, d_static=100),
                                 dict(nodes=2000, events=30000, d_e=0, d_static=0)])
def test_graph_barriers_bitwise_equal_direct(ctx, cfg):
    g = T.TemporalGraph.synthetic(ctx, T.SynthParams(nodes=cfg["nodes"], events=cfg["events"], d_e=cfg["d_e"],
                                                     seed=4))
    _, _, t = g.events()
    mc = T.ModelConfig(d_mem=100, d_time=100, d_static=cfg["d_static"], d_attn=100, d_hidden=100, d_e=cfg["d_e"],
                       n_neighbors=10, num_nodes=cfg["nodes"], max_t=float(t[-1]))
    tc = T.TrainConfig(local_batch=600, lr_base=1e-3, seed=2, epochs=2)
    res = {}
    for graphs in (True, False):
        run = T.Run(ctx, g, mc, tc, 0, cfg["events"] * 7 // 10, use_graphs=graphs)
        n = min(run.barriers, 60)
        run.step(n // 2)
        run.step(n - n // 2)  # across a re-entry of the graph pipeline (and an epoch reset)
        res[graphs] = (run.losses(), run.params())
        run.close()
    assert np.array_equal(res[True][0], res[False][0])
    assert np.array_equal(res[True][1], res[False][1])


def test_graph_bitwise_tiny_dims(ctx):
    """Tiny widths (2-column decoder halves, 3-wide attention) put GEMM outputs
    next to other writers inside one 16-byte granule: the epilogue's bulk
    tensor stores must not touch them (a graph-mode divergence caught in r01)."""
    g = T.TemporalGraph.synthetic(ctx, T.SynthParams(nodes=20, events=120, d_e=2, seed=21))
    _, _, t = g.events()
    mc = T.ModelConfig(d_mem=3, d_time=2, d_static=2, d_attn=3, d_hidden=2, d_e=2, n_neighbors=2, num_nodes=20,
                       max_t=float(t[-1]))
    tc = T.TrainConfig(local_batch=15, lr_base=1e-3, seed=3, epochs=6)
    res = {}
    for graphs in (True, False):
        for rep in range(3 if graphs else 1):
            run = T.Run(ctx, g, mc, tc, 0, 90, use_graphs=graphs)
            run.step(run.barriers)
            res[(graphs, rep)] = (run.losses(), run.params())
            run.close()
    for rep in range(3):
        assert np.array_equal(res[(True, rep)][0], res[(False, 0)][0])
        assert np.array_equal(res[(True, rep)][1], res[(False, 0)][1])


def test_oplog_matches_reference(ctx, tmp_path):
    """(1,1,1) graph-mode run: the daemon op-log (oplog.hpp) equals the reference
    run_training's, byte for byte, and passes validate_oplog."""
    from oracle import ref
    from oracle import tgnn_oracle as O
    rg = ref.RefGraph.synthetic(60, 800, d_e=4, seed=3)
    src, dst, t, ef = rg.export()
    g = T.TemporalGraph(ctx, rg.num_nodes, rg.boundary, src, dst, t, ef)
    kw = dict(d_mem=6, d_time=4, d_static=3, d_attn=5, d_hidden=4, n_neighbors=5)
    mc = T.ModelConfig(d_e=4, num_nodes=60, max_t=float(t[-1]), **kw)
    run = T.Run(ctx, g, mc, T.TrainConfig(local_batch=50, seed=3, epochs=2), 0, 600, oplog=True)
    run.step(run.barriers)
    T.write_oplog(tmp_path / "ours.oplog", run.oplog())
    run.close()
    rg.run_oplog(O.ModelConfig(d_e=4, num_nodes=60, max_t=float(t[-1]), **kw),
                 ref.train_cfg(local_batch=50, seed=3, epochs=2), 0, 600, str(tmp_path / "ref"))
    assert (tmp_path / "ours.oplog").read_text() == (tmp_path / "ref.0.oplog").read_text()
    assert ref.validate_oplog(str(tmp_path / "ours.oplog"), 1, 1)[0]
