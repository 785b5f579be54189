"""The reference-side C++ drop-in (include/tgnn_b200.hpp).

CPU: the shim compiles against the UNMODIFIED reference headers
(/root/reference/proj/include) and links libtgnn_b200.so; its host paths
(init_params, the schedule, checkpoints, error mapping) agree with the
reference's own functions. GPU: the same program runs the drop-in on cuda:0 --
sampler, plan, MemoryClient, evaluate_mrr, and run_training with the
reference's RunOptions / RunResult (op-logs byte-identical, metrics_out,
on_eval weights, segment snapshots, acceptance criterion 7 and criterion 8 on
the mean over training seeds 5..12 against tests/golden/convergence_ref.json).
The driver source is oracle/shim_driver.cpp (test infrastructure); the GPU box
has no /root/reference, so it runs the copy oracle/Makefile built here.
"""
from __future__ import annotations

import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/include"
PREBUILT = os.path.join(ROOT, "oracle", "_ref", "shim_driver")


def _compile(out):
    cmd = ["g++", "-std=c++20", "-O1", "-pthread", "-I", REF_INC, "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "oracle", "shim_driver.cpp"), "-o", out,
           "-L", os.path.join(ROOT, "paper_2307_07649_b200"), "-ltgnn_b200",
           "-Wl,-rpath," + os.path.join(ROOT, "paper_2307_07649_b200")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_INC, "tgnn")), reason="reference headers absent")
def test_shim_compiles_against_reference_and_matches_host_paths(tmp_path):
    exe = str(tmp_path / "shim_driver")
    _compile(exe)
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=300)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "cpu: 0 failure(s)" in r.stdout


@pytest.mark.gpu
def test_shim_drop_in_on_gpu():
    assert os.path.exists(PREBUILT), "oracle/_ref/shim_driver missing: run __graft_entry__.build() with the reference present"
    with open(os.path.join(ROOT, "tests", "golden", "convergence_ref.json")) as f:
        conv = json.load(f)
    means = [sum(conv[shape][str(sd)] for sd in range(5, 13)) / 8 for shape in ("1x1x1", "1x1x4")]
    r = subprocess.run([PREBUILT, "gpu"] + [f"{m:.6f}" for m in means], capture_output=True, text=True,
                       timeout=1500, cwd=ROOT)
    print(r.stdout)
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-3000:]
    assert "gpu: 0 failure(s)" in r.stdout
