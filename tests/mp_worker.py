"""torchrun worker for tests/test_multigpu.py: one rank of an i x j x k run
(one GPU per trainer), rank 0 saves barrier losses + final params."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


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
    ap.add_argument("--direct", action="store_true", help="single-stream path instead of CUDA graphs")
    a = ap.parse_args()
    import torch
    import torch.distributed as dist

    import paper_2307_07649_b200 as T
    rank, world, lr_ = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(lr_)
    dist.init_process_group("nccl", device_id=torch.device("cuda", lr_))
    s = T.gen_synthetic(T.SynthParams(nodes=20, events=120, d_e=2, seed=21))
    ctx = T.Context(lr_)
    g = T.TemporalGraph.from_stream(ctx, s)
    mc = T.ModelConfig(d_mem=3, d_time=2, d_static=2, d_attn=3, d_hidden=2, d_e=2, n_neighbors=2,
                       num_nodes=20, max_t=float(s.t[-1]))
    tc = T.TrainConfig(i=a.i, j=a.j, k=a.k, local_batch=a.local_batch, epochs=a.epochs, seed=3,
                       lr_base=a.lr)
    run = T.Run(ctx, g, mc, tc, 0, a.train_end, rank=rank, nranks=world, oplog=True, use_graphs=not a.direct)
    uid = torch.zeros(128, dtype=torch.uint8, device="cuda")
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(T.comm_unique_id()), dtype=torch.uint8))
    dist.broadcast(uid, 0)
    run.comm_init(bytes(uid.cpu().numpy().tobytes()))
    run.step(run.barriers)
    losses = run.losses()
    params = run.params()
    allp = [torch.zeros(len(params), dtype=torch.float64, device="cuda") for _ in range(world)]
    dist.all_gather(allp, torch.tensor(params, device="cuda"))
    same = all(torch.equal(allp[0], x) for x in allp)
    run.check_replicas()  # the device-side invariant (raises ProtocolError on divergence)
    logs = [None] * world
    dist.all_gather_object(logs, (rank // (a.i * a.j), run.oplog().tolist()))
    if rank == 0:
        oplog_rows = np.array([[grp] + row for grp, rows in logs for row in rows], np.int64).reshape(-1, 7)
        np.savez(a.out, losses=losses, params=params, replicas_identical=same, barriers=run.barriers,
                 oplog=oplog_rows)
    run.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
