"""CPU: the dataset files either side of the sampler (ref temporal_graph.hpp:96-279)
against the unmodified reference (oracle/_ref): write_dataset bytes, the CSV /
.meta grammar and error messages, chronological_split."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np
import pytest

import paper_2307_07649_b200 as T
from paper_2307_07649_b200 import _lib
from oracle import ref

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def _parse_error(path):
    """Our load_dataset error (parse stage, no device needed) -> (code, message)."""
    h = C.c_void_p()
    rc = _lib.lib().tgnn_graph_load_dataset(None, os.fsencode(str(path)), 3, C.byref(h))
    return rc, _lib.lib().tgnn_last_error().decode()


def _ref_error(path):
    try:
        ref.RefGraph.load_dataset(str(path))
    except ref.RefError as e:
        return e.code, e.msg
    return 0, ""


def test_write_dataset_bytes_match_reference(tmp_path):
    for kw in (dict(nodes=60, events=800, d_e=4, seed=3), dict(nodes=40, events=300, d_e=0, seed=9, bipartite=False)):
        rg = ref.RefGraph.synthetic(**kw)
        rg.write_dataset(str(tmp_path / "ref.csv"))
        src, dst, t, ef = rg.export()
        T.write_dataset(tmp_path / "ours.csv", rg.num_nodes, rg.boundary, src, dst, t, ef if kw["d_e"] else None)
        assert (tmp_path / "ours.csv").read_bytes() == (tmp_path / "ref.csv").read_bytes()
        assert (tmp_path / "ours.meta").read_bytes() == (tmp_path / "ref.meta").read_bytes()


def test_chronological_split_matches_reference():
    rg = ref.RefGraph.synthetic(60, 801, d_e=0, seed=3)
    for tf, vf in ((0.7, 0.15), (0.5, 0.25), (0.33, 0.33)):
        assert T.chronological_split(801, tf, vf) == rg.chronological_split(tf, vf)
    with pytest.raises(T.ConfigError, match="split fractions"):
        T.chronological_split(801, 0.9, 0.2)


BAD_FILES = {
    "header": ("src,dst,time\n0,1,1.0\n", "num_nodes=4\nd_e=0\n"),
    "header_width": ("src,dst,t,f0\n0,1,1.0,2\n", "num_nodes=4\nd_e=0\n"),
    "fields": ("src,dst,t\n0,1,1.0\n\n0,2\n", "num_nodes=4\n"),
    "bad_src": ("src,dst,t\n0,1,1.0\nx,1,2.0\n", "num_nodes=4\n"),
    "bad_t": ("src,dst,t\n0,1,1.0\n0,1,2.0z\n", "num_nodes=4\n"),
    "bad_feat": ("src,dst,t,f0\n0,1,1.0,0.5\n0,1,2.0,abc\n", "num_nodes=4\nd_e=1\n"),
    "range": ("src,dst,t\n0,1,1.0\n0,9,2.0\n", "num_nodes=4\n"),
    "empty": ("", "num_nodes=4\n"),
    "meta_kv": ("src,dst,t\n", "num_nodes 4\n"),
    "meta_key": ("src,dst,t\n", "num_nodes=4\ncolor=red\n"),
    "meta_nodes": ("src,dst,t\n", "# comment\nd_e=0\n"),
    "meta_num": ("src,dst,t\n", "num_nodes=4x\n"),
}


@pytest.mark.parametrize("case", sorted(BAD_FILES))
def test_parse_errors_match_reference(tmp_path, case):
    body, meta = BAD_FILES[case]
    (tmp_path / "d.csv").write_text(body)
    (tmp_path / "d.meta").write_text(meta)
    rc, msg = _parse_error(tmp_path / "d.csv")
    rrc, rmsg = _ref_error(tmp_path / "d.csv")
    assert rrc in (1, 2), (rrc, rmsg)
    assert (rc, msg) == (rrc, rmsg)


def test_missing_files_are_config_errors(tmp_path):
    rc, msg = _parse_error(tmp_path / "none.csv")
    assert rc == 1 and msg == f"cannot open dataset sidecar: {tmp_path / 'none.meta'}"
    (tmp_path / "x.meta").write_text("num_nodes=3\n")
    rc, msg = _parse_error(tmp_path / "x.csv")
    assert (rc, msg) == _ref_error(tmp_path / "x.csv")


def test_parse_error_reports_earliest_line_across_workers(tmp_path):
    rows = ["src,dst,t"] + [f"{i % 3},{3 + i % 2},{float(i)}" for i in range(5000)]
    rows[4000] = "0,1"   # line 4001
    rows[1234] = "1,x,5"  # line 1235: the reference stops here
    (tmp_path / "d.csv").write_text("\n".join(rows) + "\n")
    (tmp_path / "d.meta").write_text("num_nodes=5\nbipartite_boundary=3\n")
    rc, msg = _parse_error(tmp_path / "d.csv")
    assert (rc, msg) == _ref_error(tmp_path / "d.csv")
    assert msg.startswith("line 1235:")
