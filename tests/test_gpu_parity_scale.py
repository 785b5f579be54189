"""GPU parity at the shapes bench.py times (BASELINE configs[2] and [4]):

  C3   LastFM shape: 1,980 nodes, the full 1,293,103-event stream, no edge
       features, static memory -- hub nodes of degree ~170k;
  C5P  GDELT shape: 16,682 nodes, 186-d edge features (padded to 188 on
       device), static memory, a 1M-event prefix of the stream (the generator
       is sequential, so it IS the full stream's prefix) -- hubs of degree ~1e5.

Sampler (queries on the top-degree hubs included), negatives and plans are
bit-exact against the unmodified reference (oracle/_ref); one sub_step is held
to 1e-4 relative normwise and elementwise (elem_close: 1e-4 of each element,
floored at a tenth of the tensor's max; 5e-4 for the weight gradients, which
are long reductions with cancellation) -- except the 100-element
omega gradient, which is ill-conditioned at these time scales (1e-2 normwise,
see the test), and attn.bk, whose exact value is 0 (softmax shift invariance;
both sides are rounding noise, held absolutely). Decoder units with a hidden
pre-activation within fp32 rounding of the ReLU kink get their bias moved off
it first (clear_decoder_kinks: the gradient is discontinuous there, so fp32 and
f64 may take different branches). A 3-barrier run_sequential follows the
reference.
"""
from __future__ import annotations

import functools

import numpy as np
import pytest

import paper_2307_07649_b200 as T
from oracle import ref
from oracle import tgnn_oracle as O
from tests.helpers import REL_TOL, random_state, rel_close, tensor_slices

pytestmark = pytest.mark.gpu

C3 = dict(nodes=1980, events=1_293_103, d_e=0, seed=1)
C5P = dict(nodes=16682, events=1_000_000, d_e=186, seed=1)
MODEL = dict(d_mem=100, d_time=100, d_static=100, d_attn=100, d_hidden=100, n_neighbors=10)
CFGS = {"c3": C3, "c5p": C5P}


@functools.lru_cache(maxsize=None)
def _streams(name):
    p = CFGS[name]
    s = T.gen_synthetic(T.SynthParams(**p))
    rg = ref.RefGraph.synthetic(p["nodes"], p["events"], d_e=p["d_e"], seed=p["seed"])
    return s, rg


_G = {}


@pytest.fixture(scope="module")
def env(ctx):
    yield ctx
    for g in _G.values():
        g.close()
    _G.clear()


def setup(name, env):
    s, rg = _streams(name)
    if name not in _G:
        _G[name] = T.TemporalGraph.from_stream(env, s)
    return s, rg, _G[name]


def model_for(s):
    return T.ModelConfig(d_e=s.d_e, num_nodes=s.num_nodes, max_t=float(s.t[-1]), **MODEL)


@functools.lru_cache(maxsize=None)
def _oracle_graph(name):
    s, _ = _streams(name)
    ef = np.asarray(s.efeat, np.float64).reshape(len(s.t), -1) if s.d_e else np.zeros((len(s.t), 0))
    return O.finalize(s.num_nodes, -1, s.src, s.dst, s.t, ef)


KINK_REL = 2e-6  # 10x the distance of the flips observed at c5p@350400


def clear_decoder_kinks(name, mc, params, plan, vm, vl):
    """The decoder's ReLU (decoder.hpp:40-52) makes the gradient discontinuous
    at a zero pre-activation, and a sub-batch at these sizes has ~120k of them
    (1,200 pairs x 100 units): a handful lie within fp32 rounding of the kink
    (|pre| / (max|in| sum|W1_u|) ~ 2e-7), where the fp32 forward and the f64
    reference may take different branches -- one flip moves every upstream
    gradient by ~5e-3 relative (measured at c5p@350400: two flips, dec.b1's
    differences equal to the flips' jumps dl_e W2_u to 4 digits). So, before
    the comparison, each unit with a pre-activation within KINK_REL of the
    kink, relative to the bound max|in_e| sum|W1_u| on its terms (f64
    forward of the python oracle), has its bias dec.b1[u] moved to
    centre zero in the widest nearby gap of that unit's pre-activations --
    both sides then take the same branch everywhere. Returns (params, moved)."""
    og = _oracle_graph(name)
    omc = O.ModelConfig(**mc.__dict__)
    P = O.unflatten(omc, params)
    s_hat, _ = O.freshen(omc, P, og, vm, vl)
    h = O.embed_roots(omc, P, og, plan["root_node"], plan["root_t"], plan["supports"], s_hat)
    hs, hd, hn = h[0::3], h[1::3], h[2::3]
    inp = np.concatenate([np.concatenate([hs, hd], 1), np.concatenate([hs, hn], 1)], 0)
    W1, b1 = P["dec.W1"], P["dec.b1"].copy()
    pre = inp @ W1.T + b1
    scale = np.abs(inp).max(1)[:, None] * np.abs(W1).sum(1)[None, :]  # bound on |pre|'s terms
    moved = []
    for u in np.where((np.abs(pre) < KINK_REL * scale).any(0))[0]:
        v = np.sort(pre[:, u])
        gaps = np.diff(v)
        near = np.argsort(np.abs(0.5 * (v[1:] + v[:-1])))[:8]  # gaps close to zero
        k = near[np.argmax(gaps[near])]
        b1[u] -= 0.5 * (v[k] + v[k + 1])  # zero moves to the gap's middle
        assert 0.5 * gaps[k] > KINK_REL * scale[:, u].max()
        moved.append(int(u))
    P["dec.b1"] = b1
    return O.flatten(omc, P), moved


def elem_close(a, b, tol=REL_TOL, floor=0.1):
    """Elementwise: |a - b| <= tol * max(|b|, floor * max|b|) for EVERY element
    -- 1e-4 relative to each element of at least a tenth of the tensor's max,
    1e-5 of the max below that (values from cancellation, e.g. (1 - z) s + z h
    with s ~ -h, carry the bf16x3 GEMMs' absolute rounding, ~1e-6 of the row
    scale, which no relative bound on a tiny element can absorb). Returns
    (ok, worst ratio to the bound, worst plain relative error on |b| > 1e-3 max)."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    if not b.size or not np.abs(b).max():
        return True, 0.0, 0.0
    m = np.abs(b).max()
    bound = tol * np.maximum(np.abs(b), floor * m)
    err = np.abs(a - b)
    big = np.abs(b) > 1e-3 * m
    return bool(np.all(err <= bound)), float((err / bound).max()), float((err[big] / np.abs(b[big])).max())


@pytest.mark.parametrize("name", ["c3", "c5p"])
def test_sampler_bit_exact_with_hubs(env, name):
    s, rg, g = setup(name, env)
    deg = np.bincount(s.src, minlength=s.num_nodes) + np.bincount(s.dst, minlength=s.num_nodes)
    hubs = np.argsort(-deg)[:32]
    assert deg[hubs[0]] > 50_000, deg[hubs[0]]  # the high-degree regime this test is for
    rng = np.random.default_rng(5)
    q = 4000
    nodes = rng.integers(0, s.num_nodes, q)
    times = s.t[rng.integers(0, s.num_events, q)]
    nodes[:640] = np.repeat(hubs, 20)  # every hub at 20 times across the stream
    times[:640] = s.t[np.linspace(0, s.num_events - 1, 20).astype(np.int64)].tolist() * 32
    times[640:700] = s.t[-1] + 1.0  # past the end: the last n of the full incidence list
    for n in (10, 1):
        nn, ne, nd, cnt = g.sample_recent_neighbors_batch(nodes, times, n)
        for x in range(q):
            a = rg.sample_recent_neighbors(int(nodes[x]), float(times[x]), n)
            c = int(cnt[x])
            assert c == len(a[0]), (x, nodes[x])
            assert np.array_equal(nn[x, :c], a[0]) and np.array_equal(ne[x, :c], a[1]), (x, nodes[x])
            assert np.array_equal(nd[x, :c], a[2]), (x, nodes[x])


@pytest.mark.parametrize("name", ["c3", "c5p"])
def test_negatives_bit_exact(env, name):
    s, rg, g = setup(name, env)
    for batch, group, count, seed in [(0, 0, 600, 1), (411, 2, 1200, 1), (1500, 123456, 4800, 7)]:
        assert np.array_equal(g.sample_negatives(batch, group, count, seed),
                              rg.sample_negatives(batch, group, count, seed))


@pytest.mark.parametrize("name,begin", [("c3", 0), ("c3", 452_400), ("c3", 1_200_000), ("c5p", 350_400),
                                        ("c5p", 900_000)])
def test_plan_bit_exact(env, name, begin):
    s, rg, g = setup(name, env)
    B = 600
    negs = rg.sample_negatives(begin // B, 3, B, 1)
    a = g.plan_sub_batch(begin, begin + B, negs, 10)
    b = rg.plan_sub_batch(begin, begin + B, negs, 10)
    for k in ("root_node", "root_t", "nbr_count", "nbr_node", "nbr_event", "nbr_dt", "supports"):
        assert np.array_equal(a[k], b[k]), k


@pytest.mark.parametrize("name,begin", [("c3", 452_400), ("c5p", 350_400)])
def test_sub_step_parity_elementwise(env, name, begin):
    s, rg, g = setup(name, env)
    mc = model_for(s)
    B = 600
    rng = np.random.default_rng(1)
    params = ref.init_params(mc, 5)
    params = params + rng.normal(scale=0.02, size=params.shape) * (params != 0)
    negs = rg.sample_negatives(begin // B, 3, B, 1)
    plan = rg.plan_sub_batch(begin, begin + B, negs, mc.n_neighbors)
    st = random_state(s.num_nodes, mc.d_mem, s.t, begin, seed=1)
    vm, vl = st.read(plan["supports"])
    params, moved = clear_decoder_kinks(name, mc, params, plan, vm, vl)
    print(f"\n{name}@{begin}: decoder units moved off the ReLU kink: {moved}")
    loss_r, grads_r, shat_r = rg.sub_step(mc, params, begin, begin + B, negs, vm, vl)
    tr = T.TrainerCore(env, g, mc, B, 1)
    tr.set_params(params)
    loss, shat = tr.sub_step(begin, begin + B, negs, vm, vl)
    grads = tr.grads()
    assert abs(loss - loss_r) <= REL_TOL * abs(loss_r), (loss, loss_r)
    ok, err, sc = rel_close(shat, shat_r)
    assert ok, ("s_hat", err, sc)
    ok, worst, rel3 = elem_close(shat, shat_r)
    print(f"\n{name} s_hat: bound ratio {worst:.3g}, max rel on |x| > 1e-3 max {rel3:.3g}")
    assert ok, ("s_hat elementwise", worst)
    for tname, sl in tensor_slices(mc).items():
        # omega (d_time = 100 of the ~2M parameters) is ill-conditioned at these
        # time scales: its gradient sums per-pair terms dkv_t * (-dt sin(dt w))
        # with dt up to ~3e5 whose magnitudes cancel (sum |term| / |sum| up to
        # 1.8e3 at C5P and 1.4e3 at C3, measured on the f64 oracle; DESIGN.md
        # section 5), so the fp32 forward's ~1e-6 relative rounding of each
        # term shows up as ~5e-3 -- identically with the exact-fp32 SIMT GEMM
        # engine, i.e. it is not the tensor-core path. Stated bound: 1e-2.
        if tname == "attn.bk":
            # dL/db_k is identically 0 (adding one vector to every key of a root
            # shifts all its scores by q.b_k: softmax is invariant), so both
            # sides carry only rounding noise: held absolutely, at 1e-4 of the
            # W_k gradient's scale
            wk = tensor_slices(mc)["attn.Wk"]
            noise = np.abs(grads[sl]).max()
            print(f"{name} attn.bk: |ours| max {noise:.3g}, |ref| max {np.abs(grads_r[sl]).max():.3g}")
            assert noise <= 1e-4 * np.abs(grads_r[wk]).max()
            continue
        tol = 1e-2 if tname == "omega" else REL_TOL
        ok, err, sc = rel_close(grads[sl], grads_r[sl], tol=tol, floor=1e-7)
        assert ok, (tname, err, sc)
        # elementwise, the weight gradients (reductions over U or P rows with
        # cancellation) are held to 5e-4 of max(|x|, max/10): the exact-fp32
        # SIMT engine itself reaches 3.5e-4 on attn.Wq at c5p@900000 (the fp32
        # forward's rounding, amplified by the reduction's cancellation); omega
        # (above) is held normwise only
        ok, worst, rel3 = elem_close(grads[sl], grads_r[sl], tol=5e-4)
        print(f"{name} {tname}: normwise {err / max(sc, 1e-30):.3g}, elementwise bound ratio {worst:.3g}, "
              f"max rel on |x| > 1e-3 max {rel3:.3g}")
        assert ok or tname == "omega", (tname, "elementwise", worst)
    # root writes: nodes, t / dt / event bit-exact
    nodes_r, mem_r, mail_r = rg.build_root_writes(mc.d_mem, mc.n_neighbors, begin, begin + B, negs, vm, vl,
                                                  shat_r)
    nodes, mem, mail = tr.root_writes()
    assert np.array_equal(nodes, nodes_r)
    assert np.array_equal(mail[:, 2 * mc.d_mem:], mail_r[:, 2 * mc.d_mem:])
    assert rel_close(mem, mem_r)[0]
    tr.close()


@pytest.mark.parametrize("name,begin", [("c3", 600_000), ("c5p", 600_000)])
def test_run_sequential_three_barriers(env, name, begin):
    """run_sequential (trainer.hpp:777-867) over three mid-stream barriers
    from a fresh state: the first barrier's loss within 1e-4, the later ones
    within 1e-3, and the weights within the Adam trajectory bound."""
    s, rg, g = setup(name, env)
    mc = model_for(s)
    B = 600
    end = begin + 3 * B
    tc = T.TrainConfig(local_batch=B, seed=3, epochs=1)
    r = rg.run(mc, ref.train_cfg(local_batch=B, seed=3, epochs=1), begin, end)
    res = T.run_sequential(env, g, mc, tc, begin, end)
    assert res.barriers == r["barriers"] == 3
    # barrier 0 runs on the initial weights: the fp32 step within 1e-4; the
    # later ones follow fp32 vs f64 Adam trajectories (SURVEY 7 hard part 10)
    assert abs(res.barrier_loss[0] - r["barrier_loss"][0]) <= 1e-4 * abs(r["barrier_loss"][0])
    ok, err, sc = rel_close(res.barrier_loss, r["barrier_loss"], tol=1e-3)
    assert ok, (res.barrier_loss, r["barrier_loss"])
    lr = T.lr_eff(tc)
    assert np.abs(res.params - r["params"]).max() <= 2.5 * lr * res.barriers
    assert np.median(np.abs(res.params - r["params"])) <= 2e-5
