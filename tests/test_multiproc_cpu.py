"""CPU, world_size 2 over gloo: the host-side N>1 logic.

* every rank derives the same i x j x k schedule from build_assignment; the
  members' slices tile each global batch and activity counts agree;
* communicator bootstrap plumbing (unique-id broadcast);
* mini-batch-parallel memory semantics: two members compute root writes from
  the same pre-batch state, exchange them (all-gather) and apply in member
  order (later member wins) -- equal to replaying the whole global batch,
  the reference's invariant (ref/tests/test_trainer.cpp:190-228).
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2307_07649_b200 as T
    from oracle import tgnn_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # 1) schedule agreement
        tc = T.TrainConfig(i=2, j=1, k=1, local_batch=25, epochs=2, seed=4)
        nb, tab = T.schedule_query(tc, 0, 400, rank)
        mine = np.stack([tab["slice_begin"], tab["slice_end"], tab["batch_begin"], tab["batch_end"],
                         tab["active"], tab["active_trainers"], tab["traversed_after"]])
        allt = [None] * world
        dist.all_gather_object(allt, mine)
        a, b = allt
        assert np.array_equal(a[2:4], b[2:4]) and np.array_equal(a[5:], b[5:])
        act = a[4] == 1
        assert np.array_equal(a[1][act], b[0][act])          # member 0 ends where member 1 starts
        assert np.array_equal(a[0][act], a[2][act]) and np.array_equal(b[1][act], b[3][act])
        assert np.array_equal(a[5], a[4] + b[4])
        # 2) bootstrap: rank 0's 128-byte id reaches every rank
        obj = [os.urandom(128) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert len(obj[0]) == 128
        # 3) member writes exchanged and applied in member order == whole-batch replay
        s = T.gen_synthetic(T.SynthParams(nodes=30, events=200, d_e=2, seed=8))
        og = O.finalize(s.num_nodes, s.boundary, s.src, s.dst, s.t, s.efeat.astype(np.float64))
        mc = O.ModelConfig(d_mem=4, d_time=2, d_static=2, d_attn=3, d_hidden=3, d_e=2, n_neighbors=3,
                           num_nodes=30, max_t=float(s.t[-1]))
        params = O.init_params(mc, 1)
        state = O.MemoryState.init(30, 4)
        for lo in range(0, 120, 40):  # warm some state
            O.replay_batch(mc, params, og, state, lo, lo + 40)
        gb, ge = 120, 160
        lo, hi = (gb, gb + 20) if rank == 0 else (gb + 20, ge)
        negs = O.sample_negatives(og, 3, 3, ge - gb, 1)[lo - gb:hi - gb]
        plan = O.plan_sub_batch(og, lo, hi, negs, mc.n_neighbors)
        vm, vl = state.read(plan.supports)
        _, _, s_hat = O.sub_step(mc, params, og, plan, vm, vl)
        rows = O.build_root_writes(mc, og, plan, vm, vl, s_hat)
        allrows = [None] * world
        dist.all_gather_object(allrows, rows)
        mine_state = state.copy()
        for nodes, mrow, lrow in allrows:  # ascending member order
            mine_state.write(nodes, mrow, lrow)
        oracle = state.copy()
        O.replay_batch(mc, params, og, oracle, gb, ge)
        assert np.abs(mine_state.memory - oracle.memory).max() < 1e-12
        assert np.array_equal(mine_state.mail_event, oracle.mail_event)
        assert np.array_equal(mine_state.last_update, oracle.last_update)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - surfaced through the queue
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_world_size_2_host_logic():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
