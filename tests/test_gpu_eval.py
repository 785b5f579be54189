"""GPU parity of the validation path: evaluate_mrr and
replay_batch (trainer.hpp:336-468) on device against the unmodified reference
(oracle/_ref) and the numpy oracle; run_training's metrics rows
(trainer.hpp:725-743) and the metrics.csv format (trainer.hpp:607-618).

Distractors are integer work: bit-exact. Replayed memory is fp32 against the
f64 reference: 1e-4 relative (REL_TOL). MRR is a mean of 1/(1 + #ties-or-better)
over fp32 logits: a near-tie can flip one count, so MRR agrees to 5e-3.
"""
from __future__ import annotations

import io

import numpy as np
import pytest

import paper_2307_07649_b200 as T
from oracle import ref
from oracle import tgnn_oracle as O
from tests.helpers import random_state, rel_close

pytestmark = pytest.mark.gpu

MRR_TOL = 5e-3
SMALL = dict(nodes=60, events=800, d_e=4, seed=3)
SMALL_MODEL = dict(d_mem=6, d_time=4, d_static=3, d_attn=5, d_hidden=4, n_neighbors=5)
# a mid-size bipartite stream with static memory and 49 distractors (the reference default)
MID = dict(nodes=1500, events=24000, d_e=16, seed=11)
MID_MODEL = dict(d_mem=32, d_time=16, d_static=16, d_attn=32, d_hidden=32, n_neighbors=10)


@pytest.fixture(params=[T.GEMM_TMA, T.GEMM_SIMT], ids=["tma", "simt"])
def engine(request):
    old = T.get_gemm_impl()
    T.set_gemm_impl(request.param)
    yield request.param
    T.set_gemm_impl(old)


def _setup(ctx, cfg, mdims):
    s = T.gen_synthetic(T.SynthParams(**cfg))
    g = T.TemporalGraph.from_stream(ctx, s)
    rg = ref.RefGraph.synthetic(cfg["nodes"], cfg["events"], d_e=cfg["d_e"], seed=cfg["seed"])
    mc = T.ModelConfig(d_e=s.d_e, num_nodes=s.num_nodes, max_t=float(s.t[-1]), **mdims)
    return s, g, rg, mc


def _trained(rg, mc, epochs, end, batch):
    r = rg.run(O.ModelConfig(**mc.__dict__), ref.train_cfg(local_batch=batch, seed=3, epochs=epochs), 0, end)
    return r["params"]


@pytest.mark.parametrize("cfg,mdims,begin,end,n_neg", [
    (SMALL, SMALL_MODEL, 600, 700, 9), (MID, MID_MODEL, 20000, 20400, 49), (MID, MID_MODEL, 0, 50, 1)])
def test_eval_candidates_bit_exact(ctx, cfg, mdims, begin, end, n_neg):
    s, g, rg, mc = _setup(ctx, cfg, mdims)
    ev = T.Evaluator(ctx, g, mc, batch_size=end - begin, n_negatives=n_neg)
    got = ev.candidates(begin, end, seed=5)
    assert np.array_equal(got, rg.eval_candidates(begin, end, n_neg, 5))
    ev.close()


def test_eval_candidates_golden(ctx):
    gold = np.load("tests/golden/small.npz")
    g = T.TemporalGraph(ctx, int(gold["num_nodes"]), int(gold["boundary"]), gold["src"], gold["dst"],
                        gold["t"], gold["efeat"])
    mc = T.ModelConfig(d_e=4, num_nodes=int(gold["num_nodes"]), max_t=float(gold["t"][-1]), **SMALL_MODEL)
    ev = T.Evaluator(ctx, g, mc, batch_size=100, n_negatives=9)
    assert np.array_equal(ev.candidates(600, 700, seed=5), gold["eval_cand"])


@pytest.mark.parametrize("cfg,mdims,begin,end", [(SMALL, SMALL_MODEL, 300, 350), (MID, MID_MODEL, 15000, 15600)])
def test_replay_batch_parity(ctx, engine, cfg, mdims, begin, end):
    s, g, rg, mc = _setup(ctx, cfg, mdims)
    params = ref.init_params(mc, 7)
    st = random_state(s.num_nodes, mc.d_mem, s.t, begin, seed=2)
    sd = dict(memory=st.memory.copy(), last_update=st.last_update.copy(), mail_mem=st.mail_mem.copy(),
              mail_t=st.mail_t.copy(), mail_dt=st.mail_dt.copy(), mail_event=st.mail_event.copy())
    store = T.NodeMemoryStore(ctx, s.num_nodes, mc.d_mem)
    store.import_(sd)
    ev = T.Evaluator(ctx, g, mc, batch_size=end - begin, n_negatives=0)
    ev.replay_batch(store, params, begin, end)
    rg.replay_batch(O.ModelConfig(**mc.__dict__), params, sd, begin, end)
    got = store.export()
    for k in ("mail_event", "mail_t", "mail_dt", "last_update"):
        assert np.array_equal(got[k], sd[k]), k  # integer / f64 bookkeeping: exact
    for k in ("memory", "mail_mem"):
        ok, err, scale = rel_close(got[k], sd[k])
        assert ok, (k, err, scale)


@pytest.mark.parametrize("which", ["init", "trained"])
def test_evaluate_mrr_small(ctx, engine, which):
    gold = np.load("tests/golden/small.npz")
    g = T.TemporalGraph(ctx, int(gold["num_nodes"]), int(gold["boundary"]), gold["src"], gold["dst"],
                        gold["t"], gold["efeat"])
    mc = T.ModelConfig(d_e=4, num_nodes=int(gold["num_nodes"]), max_t=float(gold["t"][-1]), **SMALL_MODEL)
    params = gold["init_params_seed7"] if which == "init" else gold["run_params"]
    ev = T.Evaluator(ctx, g, mc, batch_size=50, n_negatives=9)
    mrr, q = ev.evaluate_mrr(params, 600, 800, seed=5)
    want = gold[f"eval_mrr_{which}"]
    assert q == int(want[1])
    assert abs(mrr - want[0]) <= MRR_TOL, (mrr, want[0])


def test_evaluate_mrr_mid(ctx, engine):
    s, g, rg, mc = _setup(ctx, MID, MID_MODEL)
    params = _trained(rg, mc, 1, 18000, 600)
    want, wq = rg.evaluate_mrr(O.ModelConfig(**mc.__dict__), params, 18000, 21000, 600, 49, 3)
    ev = T.Evaluator(ctx, g, mc, batch_size=600, n_negatives=49)
    mrr, q = ev.evaluate_mrr(params, 18000, 21000, seed=3)
    assert q == wq == 3000
    assert abs(mrr - want) <= MRR_TOL, (mrr, want)
    # deterministic: a second evaluation rebuilds the same memory and ranks
    assert ev.evaluate_mrr(None, 18000, 21000, seed=3)[0] == mrr


def test_evaluate_mrr_errors(ctx):
    s, g, rg, mc = _setup(ctx, SMALL, SMALL_MODEL)
    with pytest.raises(T.ConfigError):
        T.Evaluator(ctx, g, mc, batch_size=0, n_negatives=9)
    ev = T.Evaluator(ctx, g, mc, batch_size=50, n_negatives=9)
    with pytest.raises(T.ConfigError):
        ev.evaluate_mrr(ref.init_params(mc, 1), 700, 900, seed=1)
    with pytest.raises(T.ConfigError):
        ev.evaluate_mrr(ref.init_params(mc, 1), 500, 400, seed=1)


def test_run_metrics_rows_match_reference(ctx):
    """run_training metrics (trainer.hpp:725-743): one row per epoch-equivalent
    eval barrier; iter and traversed exact, loss and val MRR close."""
    s, g, rg, mc = _setup(ctx, SMALL, SMALL_MODEL)
    tc = T.TrainConfig(local_batch=50, seed=3, epochs=3)
    run = T.Run(ctx, g, mc, tc, 0, 600, val_begin=600, val_end=800, eval_negatives=9, eval_batch=50)
    run.step(run.barriers)
    rows = run.metrics()
    r = rg.run(O.ModelConfig(**mc.__dict__), ref.train_cfg(local_batch=50, seed=3, epochs=3), 0, 600,
               val_begin=600, val_end=800, eval_negatives=9, eval_batch=50)
    want = r["metrics"]
    assert rows.shape == want.shape == (3, 5)
    assert np.array_equal(rows[:, :2], want[:, :2])
    assert np.abs(rows[:, 2] - want[:, 2]).max() <= 1e-3
    assert np.abs(rows[:, 3] - want[:, 3]).max() <= 0.02
    assert np.all(np.diff(rows[:, 4]) >= 0) and rows[-1, 4] > 0
    # device-weights evaluation through the run handle agrees with the evaluator
    mrr, q = run.evaluate_mrr(600, 800, 50, 9, seed=3)
    ev = T.Evaluator(ctx, g, mc, batch_size=50, n_negatives=9)
    assert ev.evaluate_mrr(run.params(), 600, 800, seed=3) == (mrr, q)
    assert mrr == rows[-1, 3]
    buf = io.StringIO()
    T.write_metrics_csv(rows, buf)
    lines = buf.getvalue().splitlines()
    assert lines[0] == "iter,traversed,loss,val_mrr,elapsed_s"
    it, tr, loss, mrr_s, el = lines[1].split(",")
    assert int(it) == int(want[0, 0]) and int(tr) == int(want[0, 1])
    assert float(loss) == rows[0, 2] and float(mrr_s) == rows[0, 3] and len(el.split(".")[1]) == 3
    run.close()
