"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref,
built from /root/reference/proj/include by oracle/Makefile). Run in the
container that has /root/reference:

    make -C oracle && python tests/golden/make_golden.py

The fixtures pin the numpy oracle restatement (tests/test_oracle_golden.py)
and the host-side restatements in the product library (generator, init,
schedule) without needing the reference at test time.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402
from oracle import tgnn_oracle as O  # noqa: E402

SMALL = dict(nodes=60, events=800, d_e=4, seed=3)
MODEL = dict(d_mem=6, d_time=4, d_static=3, d_attn=5, d_hidden=4, n_neighbors=5)


def random_state(num_nodes, d_mem, t, upto, seed=0):
    rng = np.random.default_rng(seed)
    st = O.MemoryState.init(num_nodes, d_mem)
    st.memory[:] = rng.normal(scale=0.5, size=st.memory.shape)
    st.mail_mem[:] = rng.normal(scale=0.5, size=st.mail_mem.shape)
    has = rng.random(num_nodes) < 0.8
    ev = rng.integers(0, upto, has.sum())
    st.mail_event[has] = ev
    st.mail_t[has] = t[ev]
    st.mail_dt[has] = rng.random(has.sum()) * 3.0
    st.last_update[has] = st.mail_t[has]
    return st


def main():
    out = {}
    g = ref.RefGraph.synthetic(**{k: SMALL[k] for k in ("nodes", "events", "d_e", "seed")})
    src, dst, t, ef = g.export()
    out.update(num_nodes=g.num_nodes, boundary=g.boundary, src=src, dst=dst, t=t, efeat=ef)
    # a non-bipartite stream too (self-loop avoidance path of the generator)
    g2 = ref.RefGraph.synthetic(40, 300, d_e=2, seed=9, bipartite=False)
    s2, d2, t2, e2 = g2.export()
    out.update(nb_src=s2, nb_dst=d2, nb_t=t2, nb_efeat=e2)

    # sampler: queries at every 7th event time for a spread of nodes
    rng = np.random.default_rng(1)
    qn = rng.integers(0, g.num_nodes, 200)
    qt = t[rng.integers(0, len(t), 200)]
    qt[:5] = t[0]
    nbr = np.full((200, 10), -1, np.int64)
    nev = np.full((200, 10), -1, np.int64)
    ndt = np.zeros((200, 10))
    cnt = np.zeros(200, np.int64)
    for x in range(200):
        a, b, c = g.sample_recent_neighbors(int(qn[x]), float(qt[x]), 10)
        cnt[x] = len(a)
        nbr[x, :len(a)] = a
        nev[x, :len(a)] = b
        ndt[x, :len(a)] = c
    out.update(q_nodes=qn, q_times=qt, q_nbr=nbr, q_ev=nev, q_dt=ndt, q_cnt=cnt)

    neg_cases = np.array([(0, 0, 600, 1), (17, 5, 1200, 3), (3, 123456, 7, 99)], np.int64)
    for x, (b, gr, c, sd) in enumerate(neg_cases):
        out[f"negs_{x}"] = g.sample_negatives(int(b), int(gr), int(c), int(sd))
    out["neg_cases"] = neg_cases

    begin, end = 300, 350
    negs = g.sample_negatives(6, 3, end - begin, 1)
    plan = g.plan_sub_batch(begin, end, negs, MODEL["n_neighbors"])
    out["plan_negs"] = negs
    for k, v in plan.items():
        if isinstance(v, np.ndarray):
            out[f"plan_{k}"] = v

    mc = O.ModelConfig(d_e=SMALL["d_e"], num_nodes=g.num_nodes, max_t=float(t[-1]), **MODEL)
    params = ref.init_params(mc, 7)
    out["init_params_seed7"] = params
    st = random_state(g.num_nodes, mc.d_mem, t, begin)
    vm, vl = st.read(plan["supports"])
    loss, grads, s_hat = g.sub_step(mc, params, begin, end, negs, vm, vl)
    out.update(view_mem=vm, view_mail=vl, step_loss=np.array(loss), step_grads=grads,
               step_s_hat=s_hat)
    w_nodes, w_mem, w_mail = g.build_root_writes(mc.d_mem, mc.n_neighbors, begin, end, negs, vm, vl,
                                                 s_hat)
    out.update(w_nodes=w_nodes, w_mem=w_mem, w_mail=w_mail)
    adam = ref.RefAdam(len(params))
    p1 = params.copy()
    adam.step(mc, p1, grads, 1e-2)
    adam.step(mc, p1, grads, 1e-2)
    out["adam2_params"] = p1

    # replay_batch on the injected state
    sd = dict(memory=st.memory.copy(), last_update=st.last_update.copy(),
              mail_mem=st.mail_mem.copy(), mail_t=st.mail_t.copy(), mail_dt=st.mail_dt.copy(),
              mail_event=st.mail_event.copy())
    g.replay_batch(mc, params, sd, begin, end)
    for k, v in sd.items():
        out[f"replay_{k}"] = v

    # run_sequential: 2 epochs over [0, 600) in batches of 50
    r = g.run(mc, ref.train_cfg(local_batch=50, seed=3, epochs=2), 0, 600)
    out.update(run_losses=r["barrier_loss"], run_params=r["params"])

    # evaluate_mrr (trainer.hpp:383-468): distractors, and MRR of the initial
    # and of the trained weights over [600, 800) in batches of 50, 9 negatives
    out["eval_cand"] = g.eval_candidates(600, 700, 9, 5)
    out["eval_mrr_init"] = np.array(g.evaluate_mrr(mc, params, 600, 800, 50, 9, 5))
    out["eval_mrr_trained"] = np.array(g.evaluate_mrr(mc, r["params"], 600, 800, 50, 9, 5))

    # model.ckpt written by the reference's save_checkpoint (model.hpp:170-186)
    ref.save_checkpoint(mc, r["params"], os.path.join(HERE, "small.ckpt"))

    # schedules for several (i, j, k)
    shapes = np.array([(1, 1, 1, 2), (2, 1, 1, 1), (1, 2, 1, 2), (1, 1, 2, 1), (2, 2, 2, 3),
                       (1, 4, 2, 2), (1, 1, 8, 8)], np.int64)
    out["sched_shapes"] = shapes
    for x, (i, j, k, ep) in enumerate(shapes):
        a = ref.assignment(ref.train_cfg(i=int(i), j=int(j), k=int(k), local_batch=50,
                                         epochs=int(ep), seed=5), 0, 1234)
        for key in ("active", "sub", "slice_begin", "slice_end", "neg_group", "active_trainers",
                    "traversed_after", "eval_barriers"):
            out[f"sched{x}_{key}"] = a[key]

    path = os.path.join(HERE, "small.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
