"""GPU: the input pipeline -- streaming synthetic generation into
HBM, the device finalize (stable sort + validation + T-CSR) and the CSV loader --
bit-exact against the unmodified reference (oracle/_ref)."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2307_07649_b200 as T
from oracle import ref

pytestmark = pytest.mark.gpu


def _sampler_equal(g, rg, rng, q=2000, n=10):
    src, dst, t, _ = rg.export(feats=False)
    nodes = rng.integers(0, rg.num_nodes, q)
    times = t[rng.integers(0, len(t), q)] if len(t) else np.zeros(q)
    nn, ne, nd, cnt = g.sample_recent_neighbors_batch(nodes, times, n)
    for x in range(q):
        a = rg.sample_recent_neighbors(int(nodes[x]), float(times[x]), n)
        c = int(cnt[x])
        assert c == len(a[0])
        assert np.array_equal(nn[x, :c], a[0]) and np.array_equal(ne[x, :c], a[1])
        assert np.array_equal(nd[x, :c], a[2])


@pytest.mark.parametrize("kw", [dict(nodes=60, events=800, d_e=4, seed=3),
                                dict(nodes=40, events=3000, d_e=3, seed=9, bipartite=False),
                                dict(nodes=9227, events=157474, d_e=172, seed=1)])
@pytest.mark.parametrize("threads", [1, 5])
def test_streaming_synthetic_bit_exact(ctx, kw, threads):
    g = T.TemporalGraph.synthetic(ctx, T.SynthParams(**kw), threads=threads)
    rg = ref.RefGraph.synthetic(kw["nodes"], kw["events"], d_e=kw["d_e"], seed=kw["seed"],
                                bipartite=kw.get("bipartite", True))
    assert (g.num_nodes, g.boundary, g.num_events, g.d_e) == (rg.num_nodes, rg.boundary, rg.num_events, rg.d_e)
    src, dst, t = g.events()
    rs, rd, rt, ref_ef = rg.export()
    assert np.array_equal(src, rs) and np.array_equal(dst, rd) and np.array_equal(t, rt)
    assert np.array_equal(g.edge_feats(), ref_ef.astype(np.float32))
    _sampler_equal(g, rg, np.random.default_rng(1))


def test_device_finalize_sorts_stably(ctx):
    """Unsorted input with tied timestamps and self-loops: the device stable sort
    and T-CSR equal the reference finalize (temporal_graph.hpp:55-91)."""
    rng = np.random.default_rng(5)
    E, N, de = 5000, 50, 3
    src = rng.integers(0, N, E)
    dst = rng.integers(0, N, E)
    dst[:40] = src[:40]  # self-loops
    t = rng.integers(0, 300, E).astype(np.float64)  # many ties
    t[7] = -0.0
    t[8] = 0.0
    ef = rng.normal(size=(E, de))
    g = T.TemporalGraph(ctx, N, -1, src, dst, t, ef)
    rg = ref.RefGraph.from_events(N, -1, src, dst, t, ef, d_e=de)
    a = g.events()
    b = rg.export()
    for x in range(3):
        assert np.array_equal(a[x], b[x])
    assert np.array_equal(g.edge_feats(), b[3].astype(np.float32))
    _sampler_equal(g, rg, rng, q=3000)


@pytest.mark.parametrize("case", ["range", "cross"])
def test_device_finalize_errors_match_reference(ctx, case):
    src = np.array([0, 1, 2, 0, 1])
    dst = np.array([3, 4, 3, 4, 3])
    t = np.array([5.0, 1.0, 3.0, 2.0, 4.0])
    if case == "range":
        dst[2] = 7  # sorted position 2
        dst[4] = -1  # sorted position 3
    else:
        src[3], dst[3] = 3, 0  # sorted position 1 does not cross
        dst[0] = 9
    with pytest.raises(ref.RefError) as want:
        ref.RefGraph.from_events(5, 3, src, dst, t)
    with pytest.raises(T.ConfigError) as got:
        T.TemporalGraph(ctx, 5, 3, src, dst, t)
    assert str(got.value) == want.value.msg


def test_load_dataset_matches_reference(ctx, tmp_path):
    rg = ref.RefGraph.synthetic(300, 6000, d_e=5, seed=4)
    rg.write_dataset(str(tmp_path / "d.csv"))
    g = T.TemporalGraph.load_dataset(ctx, tmp_path / "d.csv", threads=4)
    back = ref.RefGraph.load_dataset(str(tmp_path / "d.csv"))
    assert (g.num_nodes, g.boundary, g.num_events, g.d_e) == (back.num_nodes, back.boundary, back.num_events,
                                                               back.d_e)
    a = g.events()
    b = back.export()
    for x in range(3):
        assert np.array_equal(a[x], b[x])
    assert np.array_equal(g.edge_feats(), b[3].astype(np.float32))
    _sampler_equal(g, back, np.random.default_rng(2))


def test_ingest_is_ordered_before_later_work(ctx):
    """tgnn_graph_ingest copies on the context's copy stream: work enqueued
    after the call must see the new rows. Overwriting a window of edge
    features and training gives bitwise the run of a graph built with them."""
    kw = dict(nodes=300, events=6000, d_e=5, seed=11)
    g1 = T.TemporalGraph.synthetic(ctx, T.SynthParams(**kw))
    src, dst, t = g1.events()
    ef = g1.edge_feats().astype(np.float64)
    a, b = 1500, 3900
    ef2 = ef.copy()
    ef2[a:b] = -0.5 * ef2[a:b] + 0.25
    g2 = T.TemporalGraph(ctx, g1.num_nodes, g1.boundary, src, dst, t, ef2)
    n = b - a
    p_src = T.pinned_empty((n,), np.int32)
    p_dst = T.pinned_empty((n,), np.int32)
    p_t = T.pinned_empty((n,), np.float64)
    p_f = T.pinned_empty((n, 5), np.float32)
    p_src[:] = src[a:b]
    p_dst[:] = dst[a:b]
    p_t[:] = t[a:b]
    p_f[:] = ef2[a:b].astype(np.float32)
    mc = T.ModelConfig(d_mem=16, d_time=8, d_static=4, d_attn=16, d_hidden=8, d_e=5, n_neighbors=5,
                       num_nodes=g1.num_nodes, max_t=float(t[-1]))
    tc = T.TrainConfig(local_batch=200, lr_base=1e-3, seed=2, epochs=1)
    res = []
    for g, ingest in ((g1, True), (g2, False)):
        if ingest:
            g.ingest(a, p_src, p_dst, p_t, p_f)  # no sync: the run below is ordered after it
        run = T.Run(ctx, g, mc, tc, 0, 4200)
        run.step(run.barriers)
        res.append((run.losses(), run.params()))
        run.close()
    assert np.array_equal(g1.edge_feats(), ef2.astype(np.float32))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])


def test_ingest_rejects_events_that_differ_from_the_index(ctx):
    """Ingested src / dst / t are verified bitwise against the finalized
    T-CSR events (never rewritten): a differing event fails the next
    synchronising call with ProtocolError and leaves the graph unchanged."""
    g = T.TemporalGraph.synthetic(ctx, T.SynthParams(nodes=50, events=400, d_e=2, seed=4))
    src, dst, t = g.events()
    a, n = 100, 20
    p_src = T.pinned_empty((n,), np.int32)
    p_dst = T.pinned_empty((n,), np.int32)
    p_t = T.pinned_empty((n,), np.float64)
    p_f = T.pinned_empty((n, 2), np.float32)
    p_src[:], p_dst[:], p_t[:] = src[a:a + n], dst[a:a + n], t[a:a + n]
    p_f[:] = g.edge_feats(a, n)
    g.ingest(a, p_src, p_dst, p_t, p_f)
    ctx.synchronize()
    for field in ("src", "t"):
        q_src, q_t = p_src.copy(), p_t.copy()
        if field == "src":
            q_src[3] = (q_src[3] + 1) % 50
        else:
            q_t[7] = np.nextafter(q_t[7], np.inf)
        b_src = T.pinned_empty((n,), np.int32)
        b_t = T.pinned_empty((n,), np.float64)
        b_src[:], b_t[:] = q_src, q_t
        g.ingest(a, b_src, p_dst, b_t, p_f)
        mc = T.ModelConfig(d_mem=4, d_time=2, d_static=0, d_attn=4, d_hidden=4, d_e=2, n_neighbors=3,
                           num_nodes=50, max_t=float(t[-1]))
        run = T.Run(ctx, g, mc, T.TrainConfig(local_batch=50, epochs=1), 0, 200)
        run.step(1)
        with pytest.raises(T.ProtocolError):
            run.losses()
        run.close()
    s2, d2, t2 = g.events()
    assert np.array_equal(s2, src) and np.array_equal(d2, dst) and np.array_equal(t2, t)
