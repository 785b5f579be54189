"""Generates tests/golden/convergence_ref.json: the unmodified reference's
(oracle/_ref) final validation MRR on its acceptance benchmark
(ref/tests/acceptance.cpp:402-458: synthetic 300-node / 5000-event graph,
d_mem 24, batch 175, lr 2e-3, 150 epochs over [0, 3500), evaluate_mrr on
[3500, 4500) with 49 negatives, eval seed 5) at several training seeds, for
the i x j x k shapes tests/test_multigpu.py checks. Seed 5 is the
reference's own (its anchors: 0.8767 / 0.8824 / 0.8368).

  python tests/golden/make_convergence_ref.py   (needs oracle/_ref built)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
import paper_2307_07649_b200 as T  # noqa: E402

SHAPES = [(1, 1, 1), (1, 1, 4), (1, 4, 1)]
SEEDS = list(range(5, 13))


def main():
    g = ref.RefGraph.synthetic(300, 5000, d_e=0, seed=20260819, pref_prob=0.95, prefs_per_src=1,
                               burst_prob=0.15, zipf_s=1.1)
    _, _, t, _ = g.export(feats=False)
    mc = T.ModelConfig(d_mem=24, d_time=8, d_static=8, d_attn=24, d_hidden=24, d_e=0, n_neighbors=8,
                       num_nodes=300, max_t=float(t[-1]))
    out = {}
    for (i, j, k) in SHAPES:
        row = {}
        for sd in SEEDS:
            tc = ref.train_cfg(i=i, j=j, k=k, local_batch=175, lr_base=2e-3, epochs=150, seed=sd)
            r = g.run(mc, tc, 0, 3500)
            mrr, _ = g.evaluate_mrr(mc, r["params"], 3500, 4500, 175, 49, 5)
            row[str(sd)] = round(mrr, 6)
            print(i, j, k, sd, row[str(sd)], flush=True)
        out[f"{i}x{j}x{k}"] = row
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "convergence_ref.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
