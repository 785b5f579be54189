"""Worker for tests/test_multigpu.py::test_convergence_matches_reference_anchors:
the reference's acceptance benchmark (ref/tests/acceptance.cpp:402-458) at an
i x j x k shape; rank 0 scores the final weights with the device evaluate_mrr
and saves the MRR. --backend nccl: one GPU per trainer under torchrun;
--backend local: every rank a thread of this process on cuda:0 (in-process hub)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rank_body(a, rank, world, device, join, seed):
    import paper_2307_07649_b200 as T
    ctx = T.Context(device)
    g = T.TemporalGraph.synthetic(ctx, T.SynthParams(nodes=300, events=5000, pref_prob=0.95, prefs_per_src=1,
                                                     burst_prob=0.15, zipf_s=1.1, d_e=0, seed=20260819))
    _, _, t = g.events()
    mc = T.ModelConfig(d_mem=24, d_time=8, d_static=8, d_attn=24, d_hidden=24, d_e=0, n_neighbors=8,
                       num_nodes=300, max_t=float(t[-1]))
    tc = T.TrainConfig(i=a.i, j=a.j, k=a.k, local_batch=175, lr_base=2e-3, epochs=a.epochs, seed=seed)
    run = T.Run(ctx, g, mc, tc, 0, 3500, rank=rank, nranks=world)
    join(run)
    run.step(run.barriers)
    out = dict(traversed=run.traversed(0, run.barriers))
    if rank == 0:
        out["mrr"], out["queries"] = run.evaluate_mrr(3500, 4500, 175, 49, seed=5)
        out["params"] = run.params()
    run.close()
    g.close()
    ctx.close()
    return out


def save(path, seeds, outs):
    np.savez(path, seeds=np.array(seeds), mrr=np.array([o["mrr"] for o in outs]),
             queries=np.array([o["queries"] for o in outs]), traversed=np.array([o["traversed"] for o in outs]),
             params=outs[0]["params"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--i", type=int, default=1)
    ap.add_argument("--j", type=int, default=1)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--epochs", type=int, default=150)
    ap.add_argument("--out", required=True)
    ap.add_argument("--seeds", default="5", help="comma-separated training seeds (the reference's is 5)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "local"])
    a = ap.parse_args()
    import paper_2307_07649_b200 as T

    world = a.i * a.j * a.k
    seeds = [int(x) for x in a.seeds.split(",")]
    if a.backend == "local":
        outs = [T.run_ranks(lambda r, hub: rank_body(a, r, world, 0, lambda run: run.local_init(hub), sd), world)[0]
                for sd in seeds]
        save(a.out, seeds, outs)
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

    outs = [rank_body(a, rank, world, lr_, join, sd) for sd in seeds]
    if rank == 0:
        save(a.out, seeds, outs)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
