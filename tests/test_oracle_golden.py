"""CPU: pins the numpy oracle restatement (oracle/tgnn_oracle.py) against golden
vectors from the unmodified reference (tests/golden/make_golden.py) and the
reference's own known-answer tests."""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import tgnn_oracle as O

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "small.npz"))
MODEL = dict(d_mem=6, d_time=4, d_static=3, d_attn=5, d_hidden=4, n_neighbors=5)


@pytest.fixture(scope="module")
def og():
    return O.finalize(int(GOLD["num_nodes"]), int(GOLD["boundary"]), GOLD["src"], GOLD["dst"],
                      GOLD["t"], GOLD["efeat"])


@pytest.fixture(scope="module")
def mc(og):
    return O.ModelConfig(d_e=og.d_e, num_nodes=og.num_nodes, max_t=float(og.t[-1]), **MODEL)


def test_rng_known_values():
    # splitmix64 reference values (public test vector for seed 0 via the +gamma step)
    assert int(O.splitmix64(np.uint64(0))) == 0xE220A8397B1DCDAF
    r = O.Rng(1)
    a = [r.next_u64() for _ in range(3)]
    r2 = O.Rng(1)
    assert a == [r2.next_u64() for _ in range(3)]
    assert int(O.hash64(1, 2)) != int(O.hash64(2, 1))


def test_toy_graph_known_answers():
    """ref/tests/test_temporal_graph.cpp:13-70."""
    g = O.finalize(5, 3, [0, 1, 0, 2, 0], [3, 3, 4, 3, 3], [1.0, 2.0, 3.0, 3.0, 5.0], np.zeros((5, 0)))
    n, e, dt = O.sample_recent_neighbors(g, 0, 5.0, 10)
    assert list(n) == [4, 3] and list(dt) == [2.0, 4.0]
    assert list(O.sample_recent_neighbors(g, 0, 5.0, 1)[0]) == [4]
    assert len(O.sample_recent_neighbors(g, 0, 1.0, 10)[0]) == 0
    negs = O.sample_negatives(g, 0, 0, 200, 7)
    assert negs.min() >= 3 and negs.max() < 5
    assert np.array_equal(O.sample_negatives(g, 0, 0, 200, 7), negs)
    assert not np.array_equal(O.sample_negatives(g, 0, 1, 200, 7), negs)
    g2 = O.finalize(4, 2, [1, 0, 1], [2, 3, 3], [5.0, 1.0, 3.0], np.zeros((3, 0)))
    assert g2.t[0] == 1.0 and g2.t[2] == 5.0
    assert len(g2.incident(1)) == 2 and len(g2.incident(0)) == 1


def test_comb_known_answer():
    """ref/tests/test_memory_store.cpp:81-107: newest t wins, ties to the larger event."""
    nodes = [1, 0, 1, 0, 2, 0]
    events = [5, 6, 7, 8, 3, 4]
    ts = [2.0, 1.0, 3.0, 1.0, 9.0, 1.0]
    kept = O.comb(nodes, events, ts)
    assert [nodes[k] for k in kept] == [0, 1, 2]
    assert [events[k] for k in kept] == [8, 7, 3]


def test_memstore_known_answer():
    """ref/tests/test_memory_store.cpp:109-139."""
    st = O.MemoryState.init(4, 2)
    st.write([1], np.array([[9.0, 8.0]]), np.array([[0.1, 0.2, 0.3, 0.4, 5.0, 4.5, 17.0]]))
    assert st.memory[1].tolist() == [9.0, 8.0] and st.mail_mem[1, 2] == 0.3
    assert st.mail_t[1] == 5.0 and st.mail_dt[1] == 4.5 and st.mail_event[1] == 17
    assert st.last_update[1] == 5.0 and st.mail_event[0] == -1
    st.reset()
    assert st.memory.sum() == 0 and st.last_update[1] == 0 and st.mail_event[1] == -1


def test_sampler_golden(og):
    for x in range(len(GOLD["q_nodes"])):
        n, e, dt = O.sample_recent_neighbors(og, int(GOLD["q_nodes"][x]), float(GOLD["q_times"][x]), 10)
        c = int(GOLD["q_cnt"][x])
        assert len(n) == c
        assert np.array_equal(n, GOLD["q_nbr"][x, :c]) and np.array_equal(e, GOLD["q_ev"][x, :c])
        assert np.array_equal(dt, GOLD["q_dt"][x, :c])


def test_negatives_golden(og):
    for x, (b, g, c, s) in enumerate(GOLD["neg_cases"]):
        assert np.array_equal(O.sample_negatives(og, int(b), int(g), int(c), int(s)), GOLD[f"negs_{x}"])


def test_plan_golden(og):
    p = O.plan_sub_batch(og, 300, 350, GOLD["plan_negs"], MODEL["n_neighbors"])
    for k in ("root_node", "root_t", "nbr_count", "nbr_node", "nbr_event", "nbr_dt", "supports"):
        assert np.array_equal(getattr(p, k), GOLD[f"plan_{k}"]), k


def test_init_golden(mc):
    assert np.array_equal(O.init_params(mc, 7), GOLD["init_params_seed7"])


def test_sub_step_golden(og, mc):
    p = O.plan_sub_batch(og, 300, 350, GOLD["plan_negs"], MODEL["n_neighbors"])
    loss, grads, s_hat = O.sub_step(mc, GOLD["init_params_seed7"], og, p, GOLD["view_mem"],
                                    GOLD["view_mail"])
    assert abs(loss - float(GOLD["step_loss"])) < 1e-12
    assert np.abs(grads - GOLD["step_grads"]).max() < 1e-12
    assert np.abs(s_hat - GOLD["step_s_hat"]).max() < 1e-12
    nodes, mem, mail = O.build_root_writes(mc, og, p, GOLD["view_mem"], GOLD["view_mail"], s_hat)
    assert np.array_equal(nodes, GOLD["w_nodes"])
    assert np.abs(mem - GOLD["w_mem"]).max() < 1e-12
    assert np.array_equal(mail, GOLD["w_mail"])


def test_adam_golden(mc):
    a = O.Adam(len(GOLD["init_params_seed7"]))
    p = GOLD["init_params_seed7"].copy()
    a.step(p, GOLD["step_grads"], 1e-2)
    a.step(p, GOLD["step_grads"], 1e-2)
    assert np.abs(p - GOLD["adam2_params"]).max() < 1e-15


def test_replay_golden(og, mc):
    st = O.MemoryState.init(og.num_nodes, mc.d_mem)
    st.memory[:] = 0
    # rebuild the injected state from the stored view is not possible; replay
    # the generator's state instead
    from tests.golden.make_golden import random_state
    st = random_state(og.num_nodes, mc.d_mem, og.t, 300)
    O.replay_batch(mc, GOLD["init_params_seed7"], og, st, 300, 350)
    assert np.abs(st.memory - GOLD["replay_memory"]).max() < 1e-12
    assert np.array_equal(st.mail_event, GOLD["replay_mail_event"])
    assert np.array_equal(st.mail_t, GOLD["replay_mail_t"])
    assert np.array_equal(st.last_update, GOLD["replay_last_update"])


def test_run_sequential_golden(og, mc):
    losses, params = O.run_sequential(mc, og, 3, 50, 1e-3, 0, 600, epochs=2)
    assert np.abs(losses - GOLD["run_losses"]).max() < 1e-10
    assert np.abs(params - GOLD["run_params"]).max() < 1e-10


def test_eval_candidates_golden(og):
    """evaluate_mrr distractors (trainer.hpp:413-423) against the reference stream."""
    assert np.array_equal(O.eval_candidates(og, 600, 700, 9, 5), GOLD["eval_cand"])
    assert not np.any(GOLD["eval_cand"] == og.dst[600:700, None])


def test_evaluate_mrr_golden(og, mc):
    """evaluate_mrr (trainer.hpp:383-468) of the initial and the trained weights."""
    for key, params in (("eval_mrr_init", GOLD["init_params_seed7"]),
                        ("eval_mrr_trained", GOLD["run_params"])):
        mrr, q = O.evaluate_mrr(mc, params, og, 600, 800, 50, 9, 5)
        assert q == int(GOLD[key][1])
        assert abs(mrr - GOLD[key][0]) < 1e-12, (key, mrr, GOLD[key][0])


def test_convergence_golden_pins_the_reference_anchors():
    """tests/golden/convergence_ref.json (the unmodified reference's final val
    MRR over training seeds 5..12, made by make_convergence_ref.py) reproduces
    the reference's own acceptance anchors at seed 5
    (ref/tests/acceptance.cpp:435-458: 0.8767, 0.8824, 0.8368), so the
    eight-seed means the GPU tests compare against come from the same runs."""
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "convergence_ref.json")) as f:
        conv = json.load(f)
    for shape, anchor in (("1x1x1", 0.8767), ("1x1x4", 0.8824), ("1x4x1", 0.8368)):
        row = conv[shape]
        assert sorted(int(k) for k in row) == list(range(5, 13))
        assert abs(row["5"] - anchor) <= 5e-5, (shape, row["5"], anchor)
