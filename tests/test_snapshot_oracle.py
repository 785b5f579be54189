"""CPU: pins the segment-snapshot oracle (acceptance criterion 4,
ref/tests/acceptance.cpp:265-328). The reference run_training's snapshots at
k = 4 with frozen weights equal a fresh-state sequential replay of the batches
each memory copy traversed since its last reset -- with the reference's own
replay_batch (0 ulp) and with the numpy restatement (oracle/tgnn_oracle.py,
1e-12). The GPU side is compared with these snapshots in
tests/test_multigpu.py::test_segment_snapshots_match_reference."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import ref
from oracle import tgnn_oracle as O

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def test_reference_snapshots_equal_fresh_replay():
    from tests.test_multigpu import snapshot_reference
    rg, mc, (meta, mem, lu) = snapshot_reference()
    assert len(meta) == 16
    src, dst, t, ef = rg.export(feats=True)
    og = O.finalize(rg.num_nodes, rg.boundary, src, dst, t, ef)
    oc = O.ModelConfig(**mc.__dict__) if not isinstance(mc, O.ModelConfig) else mc
    params0 = ref.init_params(mc, 9)
    nb, gb, k = 16, 25, 4  # 400 training events in global batches of 25, 4 segments of 4 batches
    seg_len = (nb + k - 1) // k
    segs = [(s0, min(nb, s0 + seg_len)) for s0 in range(0, nb, seg_len)]
    for (grp, sweep, seg), w_mem, w_lu in zip(meta, mem, lu):
        lo = segs[grp][0] if sweep == 0 else segs[0][0]
        st = {"memory": np.zeros((120, 6)), "last_update": np.zeros(120), "mail_mem": np.zeros((120, 12)),
              "mail_t": np.zeros(120), "mail_dt": np.zeros(120), "mail_event": np.full(120, -1, np.int64)}
        ost = O.MemoryState.init(120, 6)
        for b in range(lo, segs[seg][1]):
            rg.replay_batch(mc, params0, st, b * gb, (b + 1) * gb)
            O.replay_batch(oc, params0, og, ost, b * gb, (b + 1) * gb)
        assert np.array_equal(st["memory"], w_mem), (grp, sweep, seg)
        assert np.array_equal(st["last_update"], w_lu), (grp, sweep, seg)
        assert np.abs(ost.memory - w_mem).max() <= 1e-12, (grp, sweep, seg)
        assert np.array_equal(ost.last_update, w_lu), (grp, sweep, seg)
