"""Worker for tests/test_multigpu.py: one i x j x k run, saved by rank 0.

  --backend nccl   one process per GPU under torchrun (NCCL over NVLink)
  --backend local  every rank a thread of THIS process, all on cuda:0, joined
                   through the in-process hub (tgnn_run_local_init) -- the
                   reference's own threading model, so 1-GPU boxes run every
                   i x j x k shape too.
Saves barrier losses, final params, whether every rank's weights are bitwise
identical, and the per-memory-copy op-log rows."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rank_body(a, rank, world, device, join):
    import paper_2307_07649_b200 as T
    ctx = T.Context(device)
    if a.shape == "reddit":  # C2 dimensions: the production graph pipeline at realistic timings
        g = T.TemporalGraph.synthetic(ctx, T.SynthParams(nodes=10984, events=60000, d_e=172, seed=4))
        _, _, t = g.events()
        mc = T.ModelConfig(d_mem=100, d_time=100, d_static=100, d_attn=100, d_hidden=100, d_e=172,
                           n_neighbors=10, num_nodes=10984, max_t=float(t[-1]))
    else:
        s = T.gen_synthetic(T.SynthParams(nodes=20, events=120, d_e=2, seed=21))
        g = T.TemporalGraph.from_stream(ctx, s)
        mc = T.ModelConfig(d_mem=3, d_time=2, d_static=2, d_attn=3, d_hidden=2, d_e=2, n_neighbors=2,
                           num_nodes=20, max_t=float(s.t[-1]))
    tc = T.TrainConfig(i=a.i, j=a.j, k=a.k, local_batch=a.local_batch, epochs=a.epochs, seed=3,
                       lr_base=a.lr)
    run = T.Run(ctx, g, mc, tc, 0, a.train_end, rank=rank, nranks=world, oplog=True,
                use_graphs=not a.direct, segment_snapshots=a.snapshots)
    join(run)
    run.step(run.barriers)
    out = dict(losses=run.losses(), params=run.params(), oplog=run.oplog().tolist(),
               group=rank // (a.i * a.j), barriers=run.barriers)
    run.check_replicas()  # the device-side invariant (raises ProtocolError on divergence)
    if a.snapshots:
        out["snapshots"] = run.snapshots()
    run.close()
    g.close()
    ctx.close()
    return out


def save(a, res, same):
    oplog_rows = np.array([[r["group"]] + row for r in res for row in r["oplog"]], np.int64).reshape(-1, 7)
    extra = {}
    if a.snapshots:
        # every rank of a memory copy holds the same replica: keep member 0 of team 0's
        for r_ in range(0, len(res), a.i * a.j):
            sn = res[r_]["snapshots"]
            grp = res[r_]["group"]
            extra[f"snap_meta_{grp}"] = sn["meta"]
            extra[f"snap_mem_{grp}"] = sn["memory"]
            extra[f"snap_lu_{grp}"] = sn["last_update"]
    np.savez(a.out, losses=res[0]["losses"], params=res[0]["params"], replicas_identical=same,
             barriers=res[0]["barriers"], oplog=oplog_rows, **extra)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--i", type=int, default=1)
    ap.add_argument("--j", type=int, default=1)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--local-batch", type=int, default=15)
    ap.add_argument("--lr", type=float, default=1e-3)
    ap.add_argument("--train-end", type=int, default=90)
    ap.add_argument("--out", required=True)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "local"])
    ap.add_argument("--snapshots", action="store_true")
    ap.add_argument("--shape", default="tiny", choices=["tiny", "reddit"])
    ap.add_argument("--direct", action="store_true", help="single-stream path instead of CUDA graphs")
    a = ap.parse_args()
    import paper_2307_07649_b200 as T

    world = a.i * a.j * a.k
    if a.backend == "local":
        res = T.run_ranks(lambda r, hub: rank_body(a, r, world, 0, lambda run: run.local_init(hub)), world)
        same = all(np.array_equal(res[0]["params"], x["params"]) for x in res)
        save(a, res, same)
        return
    import torch
    import torch.distributed as dist

    rank, world, lr_ = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr_)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr_))

    def join(run):
        uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(T.comm_unique_id()), dtype=torch.uint8))
        dist.broadcast(uid, 0)
        run.comm_init(bytes(uid.cpu().numpy().tobytes()))

    mine = rank_body(a, rank, world, lr_, join)
    res = [None] * world
    dist.all_gather_object(res, mine)
    if rank == 0:
        same = all(np.array_equal(res[0]["params"], x["params"]) for x in res)
        save(a, res, same)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
