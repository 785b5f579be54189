"""B200-native DistTGL training step (arXiv 2307.07649), host-side mirror.

Python view of the C ABI (include/tgnn_b200.h) with the reference's own names
and argument meanings (/root/reference/proj/include/tgnn):

  gen_synthetic                  synthetic.hpp:54-112
  TemporalGraph (finalize)       temporal_graph.hpp:33-95
    .sample_recent_neighbors     temporal_graph.hpp:296-318
    .sample_negatives            temporal_graph.hpp:355-370
    .plan_sub_batch              trainer.hpp:76-106
  NodeMemoryStore (MemoryClient) memory_store.hpp:16-50, shared_buffers.hpp:124-165
  init_params / param_count      model.hpp:122-141, optimizer.hpp:12-17
  TrainerCore                    trainer.hpp:490-562 (sub_step, build_root_writes, Adam)
  Run / run_sequential           trainer.hpp:630-867

All compute runs in libtgnn_b200.so (sm_100a CUDA kernels + NCCL); a missing
library raises at import time -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field

import numpy as np

from ._lib import (ConfigError, CudaError, ModelConfigC, NcclError, NumericError, ParseError,
                   ProtocolError, RunOptionsC, ShapeError, SynthParamsC, TgnnError, TrainConfigC,
                   check, f32p, f64p, i64p, lib)

__all__ = [
    "ConfigError", "ParseError", "NumericError", "ProtocolError", "ShapeError", "CudaError",
    "NcclError", "TgnnError", "ModelConfig", "TrainConfig", "SynthParams", "EventStream",
    "gen_synthetic", "Context", "TemporalGraph", "NodeMemoryStore", "ReadView", "TrainerCore",
    "Run", "run_sequential", "param_count", "init_params", "lr_eff", "Evaluator",
    "write_metrics_csv", "save_checkpoint", "load_checkpoint", "write_dataset", "chronological_split",
    "write_oplog", "LocalHub", "run_ranks",
]

lib()  # fail loudly at import if the native library is absent


def _p(a, t):
    return a.ctypes.data_as(t) if a is not None else None


# ---------------------------------------------------------------- configs
@dataclass
class ModelConfig:
    """ModelConfig, ref model.hpp:19-35."""

    d_mem: int = 100
    d_time: int = 100
    d_static: int = 100
    d_attn: int = 100
    d_hidden: int = 0
    d_e: int = 0
    n_neighbors: int = 10
    num_nodes: int = 0
    max_t: float = 1.0

    def c(self) -> ModelConfigC:
        return ModelConfigC(self.d_mem, self.d_time, self.d_static, self.d_attn, self.d_hidden,
                            self.d_e, self.n_neighbors, self.num_nodes, self.max_t)


@dataclass
class TrainConfig:
    """TrainConfig, ref parallel.hpp:15-50."""

    i: int = 1
    j: int = 1
    k: int = 1
    p: int = 1
    q: int = 0  # 0: i*j*k/p
    local_batch: int = 600
    lr_base: float = 1e-3
    epochs: int = 1
    seed: int = 1
    local_batch_ref: int = 0
    neg_groups: int = 0

    def c(self) -> TrainConfigC:
        q = self.q or (self.i * self.j * self.k) // self.p
        return TrainConfigC(self.i, self.j, self.k, self.p, q, self.epochs, self.local_batch,
                            self.lr_base, self.seed, self.local_batch_ref, self.neg_groups)

    @property
    def num_trainers(self) -> int:
        return self.i * self.j * self.k


def lr_eff(t: TrainConfig) -> float:
    """TrainConfig::lr_eff, ref parallel.hpp:30-34."""
    ref = t.local_batch_ref if t.local_batch_ref > 0 else t.local_batch
    return t.lr_base * (t.num_trainers * t.local_batch) / ref


@dataclass
class SynthParams:
    """SynthParams, ref synthetic.hpp:14-25."""

    nodes: int = 1000
    events: int = 10000
    burst_prob: float = 0.2
    pref_prob: float = 0.85
    prefs_per_src: int = 3
    src_frac: float = 0.5
    bipartite: bool = True
    d_e: int = 0
    zipf_s: float = 1.0
    seed: int = 1


@dataclass
class EventStream:
    num_nodes: int
    boundary: int
    src: np.ndarray
    dst: np.ndarray
    t: np.ndarray
    efeat: np.ndarray  # float32 [E, d_e]

    @property
    def d_e(self):
        return self.efeat.shape[1]

    @property
    def num_events(self):
        return len(self.t)


def _synth_c(p: SynthParams) -> SynthParamsC:
    return SynthParamsC(p.nodes, p.events, p.burst_prob, p.pref_prob, p.prefs_per_src, p.src_frac,
                        1 if p.bipartite else 0, p.d_e, p.zipf_s, p.seed)


def gen_synthetic(p: SynthParams, with_features: bool = True) -> EventStream:
    """Bit-identical host restatement of gen_synthetic (synthetic.hpp:54-112)."""
    E = int(p.events)
    src = np.empty(E, np.int64)
    dst = np.empty(E, np.int64)
    t = np.empty(E, np.float64)
    ef = np.empty((E, p.d_e), np.float32) if with_features else np.zeros((E, 0), np.float32)
    sp = SynthParamsC(p.nodes, p.events, p.burst_prob, p.pref_prob, p.prefs_per_src, p.src_frac,
                      1 if p.bipartite else 0, p.d_e, p.zipf_s, p.seed)
    b = C.c_int64()
    check(lib().tgnn_gen_synthetic(C.byref(sp), _p(src, i64p), _p(dst, i64p), _p(t, f64p),
                                   _p(ef, f32p) if with_features and p.d_e else None,
                                   C.byref(b)))
    return EventStream(int(p.nodes), b.value, src, dst, t, ef)


def param_count(m: ModelConfig) -> int:
    out = C.c_int64()
    mc = m.c()
    check(lib().tgnn_param_count(C.byref(mc), C.byref(out)))
    return out.value


def init_params(m: ModelConfig, seed: int) -> np.ndarray:
    """init_params (model.hpp:122-141), canonical flat order (model.hpp:56-76)."""
    out = np.empty(param_count(m), np.float64)
    mc = m.c()
    check(lib().tgnn_init_params(C.byref(mc), seed, _p(out, f64p)))
    return out


# ---------------------------------------------------------------- handles
class Context:
    """One CUDA device + stream (one per host thread / rank)."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(lib().tgnn_ctx_create(device, C.byref(self.h)))
        self.device = device
        self._children = []

    def _adopt(self, obj):
        """Handles created on this context are closed (newest first) before it."""
        self._children.append(weakref.ref(obj))

    def synchronize(self):
        check(lib().tgnn_ctx_synchronize(self.h))

    @property
    def stream_ptr(self) -> int:
        s = C.c_void_p()
        check(lib().tgnn_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def close(self):
        if self.h:
            for ref_ in reversed(self._children):
                obj = ref_()
                if obj is not None:
                    try:
                        obj.close()
                    except Exception:
                        pass
            self._children = []
            lib().tgnn_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TemporalGraph:
    """Device-resident TemporalGraph: events + T-CSR + fp32 edge features."""

    def __init__(self, ctx: Context, num_nodes, boundary, src, dst, t, efeat=None):
        self.ctx = ctx
        ctx._adopt(self)
        src = np.ascontiguousarray(src, np.int64)
        dst = np.ascontiguousarray(dst, np.int64)
        t = np.ascontiguousarray(t, np.float64)
        self.h = C.c_void_p()
        if efeat is None:
            efeat = np.zeros((len(t), 0), np.float32)
        d_e = efeat.shape[1] if efeat.ndim == 2 else 0
        if efeat.dtype == np.float64:
            ef = np.ascontiguousarray(efeat)
            check(lib().tgnn_graph_create_f64(ctx.h, num_nodes, boundary, len(t), _p(src, i64p),
                                              _p(dst, i64p), _p(t, f64p), _p(ef, f64p), d_e,
                                              C.byref(self.h)))
        else:
            ef = np.ascontiguousarray(efeat, np.float32)
            check(lib().tgnn_graph_create(ctx.h, num_nodes, boundary, len(t), _p(src, i64p),
                                          _p(dst, i64p), _p(t, f64p), _p(ef, f32p), d_e,
                                          C.byref(self.h)))
        self._info()

    def _info(self):
        n, b, e, de = (C.c_int64() for _ in range(4))
        check(lib().tgnn_graph_info(self.h, C.byref(n), C.byref(b), C.byref(e), C.byref(de)))
        self.num_nodes, self.boundary, self.num_events, self.d_e = n.value, b.value, e.value, de.value

    @classmethod
    def _from_handle(cls, ctx: Context, h) -> "TemporalGraph":
        g = cls.__new__(cls)
        g.ctx, g.h = ctx, h
        ctx._adopt(g)
        g._info()
        return g

    @staticmethod
    def from_stream(ctx: Context, s: EventStream) -> "TemporalGraph":
        return TemporalGraph(ctx, s.num_nodes, s.boundary, s.src, s.dst, s.t, s.efeat)

    @staticmethod
    def synthetic(ctx: Context, p: SynthParams, threads: int = 0) -> "TemporalGraph":
        """gen_synthetic (synthetic.hpp:54-112) streamed into HBM chunk by chunk,
        then finalized on the device (bit-identical to the reference stream)."""
        h = C.c_void_p()
        check(lib().tgnn_graph_synthetic(ctx.h, C.byref(_synth_c(p)), threads, C.byref(h)))
        return TemporalGraph._from_handle(ctx, h)

    @staticmethod
    def load_dataset(ctx: Context, csv_path, threads: int = 0) -> "TemporalGraph":
        """load_dataset (temporal_graph.hpp:255-258): event CSV + .meta sidecar."""
        h = C.c_void_p()
        check(lib().tgnn_graph_load_dataset(ctx.h if ctx is not None else None, os.fsencode(csv_path),
                                             threads, C.byref(h)))
        return TemporalGraph._from_handle(ctx, h)

    def edge_feats(self, first: int = 0, count=None):
        """fp32 edge-feature rows [first, first + count) (temporal_graph.hpp:46-48)."""
        count = self.num_events - first if count is None else count
        out = np.zeros((count, self.d_e), np.float32)
        check(lib().tgnn_graph_edge_feats(self.h, first, count, _p(out, f32p)))
        return out

    def bipartite(self) -> bool:
        return self.boundary >= 0

    def events(self):
        E = self.num_events
        src = np.empty(E, np.int64)
        dst = np.empty(E, np.int64)
        t = np.empty(E, np.float64)
        check(lib().tgnn_graph_events(self.h, _p(src, i64p), _p(dst, i64p), _p(t, f64p)))
        return src, dst, t

    def sample_recent_neighbors_batch(self, nodes, times, n):
        nodes = np.ascontiguousarray(nodes, np.int64)
        times = np.ascontiguousarray(times, np.float64)
        q = len(nodes)
        nn = np.empty((q, n), np.int64)
        ne = np.empty((q, n), np.int64)
        nd = np.empty((q, n), np.float64)
        cnt = np.empty(q, np.int64)
        check(lib().tgnn_sample_recent_neighbors(self.h, _p(nodes, i64p), _p(times, f64p), q, n,
                                                 _p(nn, i64p), _p(ne, i64p), _p(nd, f64p),
                                                 _p(cnt, i64p)))
        return nn, ne, nd, cnt

    def sample_recent_neighbors(self, v, t, n):
        nn, ne, nd, cnt = self.sample_recent_neighbors_batch([v], [t], n)
        c = int(cnt[0])
        return nn[0, :c], ne[0, :c], nd[0, :c]

    def sample_negatives(self, batch_index, group, count, seed):
        out = np.empty(count, np.int64)
        check(lib().tgnn_sample_negatives(self.h, batch_index, group, count, seed, _p(out, i64p)))
        return out

    def plan_sub_batch(self, begin, end, negatives, n):
        B = end - begin
        R = 3 * B
        negatives = np.ascontiguousarray(negatives, np.int64)
        rn = np.empty(R, np.int64)
        rt = np.empty(R, np.float64)
        cnt = np.empty(R, np.int64)
        nn = np.full((R, n), -1, np.int64)
        ne = np.full((R, n), -1, np.int64)
        nd = np.zeros((R, n), np.float64)
        sup = np.empty(max(R * (n + 1), 1), np.int64)
        U = C.c_int64()
        check(lib().tgnn_plan_sub_batch(self.h, begin, end, _p(negatives, i64p), n, _p(rn, i64p),
                                        _p(rt, f64p), _p(cnt, i64p), _p(nn, i64p), _p(ne, i64p),
                                        _p(nd, f64p), _p(sup, i64p), C.byref(U)))
        return dict(begin=begin, end=end, root_node=rn, root_t=rt, nbr_count=cnt, nbr_node=nn,
                    nbr_event=ne, nbr_dt=nd, supports=sup[:U.value].copy())

    def ingest(self, first, src32, dst32, t, efeat32):
        """Streams events [first, first+len) from (ideally pinned) host buffers."""
        check(lib().tgnn_graph_ingest(self.h, first, len(t), src32.ctypes.data_as(C.POINTER(C.c_int32)),
                                      dst32.ctypes.data_as(C.POINTER(C.c_int32)), _p(t, f64p),
                                      _p(efeat32, f32p) if efeat32 is not None and efeat32.size else None))

    def close(self):
        if self.h:
            lib().tgnn_graph_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class ReadView:
    """ReadView, ref shared_buffers.hpp:118-122."""

    nodes: np.ndarray
    mem: np.ndarray
    mail: np.ndarray


class NodeMemoryStore:
    """HBM-resident NodeMemoryState with the MemoryClient interface."""

    def __init__(self, ctx: Context, num_nodes: int, d_mem: int):
        self.ctx = ctx
        ctx._adopt(self)
        self.num_nodes, self.d_mem = num_nodes, d_mem
        self.h = C.c_void_p()
        check(lib().tgnn_memstore_create(ctx.h, num_nodes, d_mem, C.byref(self.h)))

    def reset(self):
        check(lib().tgnn_memstore_reset(self.h))

    def read(self, subs):
        out = []
        d = self.d_mem
        for nodes in subs:
            nodes = np.ascontiguousarray(nodes, np.int64)
            mem = np.empty((len(nodes), d), np.float64)
            mail = np.empty((len(nodes), 2 * d + 3), np.float64)
            check(lib().tgnn_memstore_read(self.h, _p(nodes, i64p), len(nodes), _p(mem, f64p),
                                           _p(mail, f64p)))
            out.append(ReadView(nodes.copy(), mem, mail))
        return out

    def write(self, nodes, mem_rows, mail_rows):
        nodes = np.ascontiguousarray(nodes, np.int64)
        mem_rows = np.ascontiguousarray(mem_rows, np.float64)
        mail_rows = np.ascontiguousarray(mail_rows, np.float64)
        check(lib().tgnn_memstore_write(self.h, _p(nodes, i64p), len(nodes), _p(mem_rows, f64p),
                                        _p(mail_rows, f64p)))

    def export(self):
        N, d = self.num_nodes, self.d_mem
        st = dict(memory=np.empty((N, d)), last_update=np.empty(N), mail_mem=np.empty((N, 2 * d)),
                  mail_t=np.empty(N), mail_dt=np.empty(N), mail_event=np.empty(N, np.int64))
        check(lib().tgnn_memstore_export(self.h, _p(st["memory"], f64p), _p(st["last_update"], f64p),
                                         _p(st["mail_mem"], f64p), _p(st["mail_t"], f64p),
                                         _p(st["mail_dt"], f64p), _p(st["mail_event"], i64p)))
        return st

    def import_(self, st):
        a = {k: np.ascontiguousarray(v, np.int64 if k == "mail_event" else np.float64)
             for k, v in st.items()}
        check(lib().tgnn_memstore_import(self.h, _p(a["memory"], f64p), _p(a["last_update"], f64p),
                                         _p(a["mail_mem"], f64p), _p(a["mail_t"], f64p),
                                         _p(a["mail_dt"], f64p), _p(a["mail_event"], i64p)))

    def close(self):
        if self.h:
            lib().tgnn_memstore_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class TrainerCore:
    """Trainer replica on one GPU: params/grads/Adam state + step workspace."""

    def __init__(self, ctx: Context, g: TemporalGraph, model: ModelConfig, max_local_batch: int,
                 seed: int):
        self.ctx, self.g, self.model, self.seed = ctx, g, model, seed
        ctx._adopt(self)
        if model.num_nodes == 0:
            model.num_nodes = g.num_nodes
        self.h = C.c_void_p()
        mc = model.c()
        check(lib().tgnn_trainer_create(ctx.h, g.h, C.byref(mc), max_local_batch, seed,
                                        C.byref(self.h)))
        self.nparam = param_count(model)
        self._U = None

    def set_params(self, flat):
        flat = np.ascontiguousarray(flat, np.float64)
        check(lib().tgnn_trainer_set_params(self.h, _p(flat, f64p)))

    def loss_async(self, b, dst):
        """Enqueues the D2H copy of this rank's barrier-b loss into dst (a pinned
        float64 array view of length >= 1); valid after the next synchronisation."""
        check(lib().tgnn_run_loss_async(self.h, b, _p(dst, f64p)))

    def params(self):
        out = np.empty(self.nparam)
        check(lib().tgnn_trainer_get_params(self.h, _p(out, f64p)))
        return out

    def grads(self):
        out = np.empty(self.nparam)
        check(lib().tgnn_trainer_get_grads(self.h, _p(out, f64p)))
        return out

    def sub_step(self, begin, end, negatives, view_mem, view_mail, want_s_hat=True):
        negatives = np.ascontiguousarray(negatives, np.int64)
        vm = np.ascontiguousarray(view_mem, np.float64)
        vl = np.ascontiguousarray(view_mail, np.float64)
        loss = C.c_double()
        sh = np.empty((vm.shape[0], self.model.d_mem)) if want_s_hat else None
        check(lib().tgnn_trainer_sub_step(self.h, begin, end, _p(negatives, i64p), _p(vm, f64p),
                                          _p(vl, f64p), C.byref(loss), _p(sh, f64p)))
        self._B = end - begin
        return loss.value, sh

    def root_writes(self):
        B = self._B
        d = self.model.d_mem
        nodes = np.empty(2 * B, np.int64)
        mem = np.empty((2 * B, d))
        mail = np.empty((2 * B, 2 * d + 3))
        W = C.c_int64()
        check(lib().tgnn_trainer_root_writes(self.h, _p(nodes, i64p), _p(mem, f64p),
                                             _p(mail, f64p), C.byref(W)))
        w = W.value
        return nodes[:w].copy(), mem[:w].copy(), mail[:w].copy()

    def adam_step(self, lr):
        check(lib().tgnn_trainer_adam_step(self.h, lr))

    def iterate(self, store: NodeMemoryStore, batch_index, group, batch_begin, begin, end, lr):
        loss = C.c_double()
        check(lib().tgnn_trainer_iterate(self.h, store.h, batch_index, group, batch_begin, begin,
                                         end, lr, C.byref(loss)))
        return loss.value

    def close(self):
        if self.h:
            lib().tgnn_trainer_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def pinned_empty(shape, dtype):
    """numpy array over page-locked host memory (freed with the array's owner)."""
    dtype = np.dtype(dtype)
    n = int(np.prod(shape)) * dtype.itemsize
    ptr = C.c_void_p()
    check(lib().tgnn_pinned_alloc(max(n, 1), C.byref(ptr)))
    buf = (C.c_char * max(n, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)
    _PINNED.append((ptr, arr))
    return arr


_PINNED = []


SCHEDULE_FIELDS = ["active", "sub", "subs", "batch", "batch_begin", "batch_end", "slice_begin",
                   "slice_end", "neg_group", "reset_before", "active_trainers", "traversed_after"]


def schedule_query(train: TrainConfig, train_begin: int, train_end: int, rank: int, first: int = 0,
                   count=None):
    """Per-barrier task table of `rank` (build_assignment + Assignment::task,
    ref parallel.hpp:150-331). Returns (barriers, dict of int64 arrays)."""
    tc = train.c()
    nb = C.c_int64()
    out = np.zeros((1, 12), np.int64)
    check(lib().tgnn_schedule_query(C.byref(tc), train_begin, train_end, rank, 0, 0, _p(out, i64p),
                                    C.byref(nb)))
    count = nb.value - first if count is None else count
    out = np.zeros((max(count, 1), 12), np.int64)
    check(lib().tgnn_schedule_query(C.byref(tc), train_begin, train_end, rank, first, count,
                                    _p(out, i64p), C.byref(nb)))
    return nb.value, {k: out[:count, x].copy() for x, k in enumerate(SCHEDULE_FIELDS)}


GEMM_SIMT, GEMM_TMA, GEMM_GATHER = 0, 1, 2
GEMM_TENSOR = GEMM_TMA


def set_gemm_impl(impl: int):
    """0: exact fp32 CUDA-core GEMMs; 1 (default): TMA-fed tcgen05 bf16x3 GEMMs over
    pre-split operands; 2: tcgen05 bf16x3 gathering fp32 operands in the GEMM."""
    check(lib().tgnn_set_gemm_impl(impl))


def get_gemm_impl() -> int:
    v = C.c_int()
    check(lib().tgnn_get_gemm_impl(C.byref(v)))
    return v.value


def debug_gemm(A, B, impl=GEMM_TMA, a_trans=False, b_trans=False, splits=1):
    """C = op(A) op(B) on device (test hook for the GEMM engines)."""
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    M = A.shape[1] if a_trans else A.shape[0]
    K = A.shape[0] if a_trans else A.shape[1]
    N = B.shape[0] if b_trans else B.shape[1]
    out = np.empty((M, N), np.float32)
    check(lib().tgnn_debug_gemm(impl, M, N, K, _p(A, f32p), int(a_trans), _p(B, f32p), int(b_trans),
                                _p(out, f32p), splits))
    return out


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().tgnn_comm_unique_id(buf))
    return buf.raw


class LocalHub:
    """In-process exchange for the ranks of one job run as threads of this
    process (tgnn_local_hub): collectives are host rendezvous + cross-stream
    events + ascending-rank device reductions, on one GPU or several."""

    def __init__(self, nranks: int):
        self.h = C.c_void_p()
        check(lib().tgnn_local_hub_create(nranks, C.byref(self.h)))
        self.nranks = nranks

    def close(self):
        if self.h:
            lib().tgnn_local_hub_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def run_ranks(fn, nranks: int, timeout: float = 900.0):
    """Runs fn(rank, hub) on nranks threads sharing one LocalHub; returns the
    per-rank results (re-raises the first failure)."""
    import threading

    hub = LocalHub(nranks)
    out, err = [None] * nranks, [None] * nranks

    def body(r):
        try:
            out[r] = fn(r, hub)
        except BaseException as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout)
    if any(t.is_alive() for t in th):
        raise TimeoutError("run_ranks: a rank did not finish")
    first = next((e for e in err if e is not None), None)
    if first is not None:
        raise first
    hub.close()
    return out


class Run:
    """One rank of run_training (trainer.hpp:630-772); nranks == i*j*k, one GPU each."""

    def __init__(self, ctx: Context, g: TemporalGraph, model: ModelConfig, train: TrainConfig,
                 train_begin: int, train_end: int, rank: int = 0, nranks: int = 1,
                 use_graphs: bool = True, val_begin: int = 0, val_end: int = 0,
                 eval_negatives: int = 49, eval_batch: int = 0, oplog: bool = False,
                 segment_snapshots: bool = False):
        self.ctx, self.g, self.model, self.train = ctx, g, model, train
        ctx._adopt(self)
        if model.num_nodes == 0:
            model.num_nodes = g.num_nodes
        opt = RunOptionsC(model.c(), train.c(), train_begin, train_end, rank, nranks,
                          1 if use_graphs else 0, val_begin, val_end, eval_negatives, 0, eval_batch,
                          1 if oplog else 0, 1 if segment_snapshots else 0)
        self.h = C.c_void_p()
        check(lib().tgnn_run_create(ctx.h, g.h, C.byref(opt), C.byref(self.h)))
        b, n = C.c_int64(), C.c_int64()
        check(lib().tgnn_run_info(self.h, C.byref(b), C.byref(n)))
        self.barriers, self.nparam = b.value, n.value
        self.rank, self.nranks = rank, nranks
        self.next = 0

    def comm_init(self, uid: bytes):
        check(lib().tgnn_run_comm_init(self.h, uid))

    def local_init(self, hub: "LocalHub"):
        """Joins the in-process hub (every rank a thread of this process); call
        from each rank's own thread -- it returns once all ranks attached."""
        check(lib().tgnn_run_local_init(self.h, hub.h))
        self.hub = hub

    def step(self, count: int = 1):
        check(lib().tgnn_run_barriers(self.h, self.next, count))
        self.next += count

    def losses(self, first=0, count=None):
        count = self.next - first if count is None else count
        out = np.empty(count)
        check(lib().tgnn_run_losses(self.h, first, count, _p(out, f64p)))
        return out

    def loss_async(self, b, dst):
        """Enqueues the D2H copy of this rank's barrier-b loss into dst (a pinned
        float64 array view of length >= 1); valid after the next synchronisation."""
        check(lib().tgnn_run_loss_async(self.h, b, _p(dst, f64p)))

    def params(self):
        out = np.empty(self.nparam)
        check(lib().tgnn_run_params(self.h, _p(out, f64p)))
        return out

    def traversed(self, first, count):
        out = C.c_int64()
        check(lib().tgnn_run_traversed(self.h, first, count, C.byref(out)))
        return out.value

    def eval_barriers(self):
        """Assignment::eval_barriers (parallel.hpp:316-329)."""
        n = C.c_int64()
        check(lib().tgnn_run_eval_barriers(self.h, C.byref(n), None))
        out = np.zeros(n.value, np.int64)
        if n.value:
            check(lib().tgnn_run_eval_barriers(self.h, C.byref(n), _p(out, i64p)))
        return out

    def metrics(self):
        """MetricsRow list (trainer.hpp:562-570) for the eval barriers run so far:
        [rows x 5] = iter, traversed, loss, val_mrr, elapsed_s. Collective at nranks > 1."""
        n = C.c_int64()
        check(lib().tgnn_run_metrics(self.h, C.byref(n), None))
        out = np.zeros((n.value, 5))
        if n.value:
            check(lib().tgnn_run_metrics(self.h, C.byref(n), _p(out, f64p)))
        return out

    def check_replicas(self) -> int:
        """Collective: raises ProtocolError unless every rank holds bitwise the
        same parameters; returns the 64-bit fingerprint."""
        h = C.c_uint64()
        check(lib().tgnn_run_check_replicas(self.h, C.byref(h)))
        return h.value

    def oplog(self):
        """This rank's daemon op-log rows [n x 6]: epoch, iter, kind (0 R / 1 W),
        rank within the memory copy, first, len (OpRecord, oplog.hpp:15-24)."""
        n = C.c_int64()
        check(lib().tgnn_run_oplog(self.h, C.byref(n), None))
        out = np.zeros((n.value, 6), np.int64)
        if n.value:
            check(lib().tgnn_run_oplog(self.h, C.byref(n), _p(out, i64p)))
        return out

    def snapshots(self):
        """RunResult.snapshots of this rank's memory copy (trainer.hpp:593):
        dict(meta [n x 2] = sweep, segment; memory [n, N, d_mem]; last_update [n, N])."""
        n = C.c_int64()
        check(lib().tgnn_run_snapshots(self.h, C.byref(n), None, None, None))
        N, d = self.g.num_nodes, self.model.d_mem
        meta = np.zeros((n.value, 2), np.int64)
        mem = np.zeros((n.value, N, d))
        lu = np.zeros((n.value, N))
        if n.value:
            check(lib().tgnn_run_snapshots(self.h, C.byref(n), _p(meta, i64p), _p(mem, f64p), _p(lu, f64p)))
        return dict(meta=meta, memory=mem, last_update=lu)

    def save_checkpoint(self, path):
        """model.ckpt of this rank's current weights (all replicas are identical)."""
        save_checkpoint(self.model, self.params(), path)

    def write_metrics_csv(self, path_or_file):
        """metrics.csv in the reference format (trainer.hpp:607-618)."""
        write_metrics_csv(self.metrics(), path_or_file)

    def evaluate_mrr(self, eval_begin: int, eval_end: int, batch_size: int, n_negatives: int = 49,
                     seed: int = 1):
        """evaluate_mrr (trainer.hpp:383-468) of this rank's current device weights."""
        mrr, q = C.c_double(), C.c_int64()
        check(lib().tgnn_run_evaluate_mrr(self.h, eval_begin, eval_end, batch_size, n_negatives, seed,
                                          C.byref(mrr), C.byref(q)))
        return mrr.value, q.value

    PHASES = ["plan", "gru_fwd", "attn_assemble", "attn_proj", "attn_softmax", "decoder",
              "decoder_bwd", "attn_bwd", "attn_bwd_gemm", "gru_bwd", "writes", "allreduce", "adam"]

    def profile_barrier(self, direct: bool = True):
        """Runs the next barrier with phase markers: ({phase: ms}, plan sizes).
        direct: the single-stream path (every phase timed alone); otherwise the
        production graph schedule (markers on the critical-path stream)."""
        ms = np.zeros(len(self.PHASES))
        sz = np.zeros(8, np.int32)
        check(lib().tgnn_run_profile_barrier(self.h, _p(ms, f64p), sz.ctypes.data_as(C.POINTER(C.c_int32)),
                                             1 if direct else 0))
        self.next += 1
        return dict(zip(self.PHASES, ms.tolist())), dict(B=int(sz[0]), R=int(sz[1]), P=int(sz[2]),
                                                         U=int(sz[3]), W=int(sz[7]))

    def gemm_profile(self):
        """Runs the next barrier (direct path) with every tcgen05 GEMM launch
        event-timed: array [launches x 6] = ms, algorithmic FLOPs, algorithmic
        bytes, problems, max M, max splits."""
        rows = np.zeros((64, 6))
        n = C.c_int64()
        check(lib().tgnn_run_gemm_profile(self.h, 64, C.byref(n), _p(rows, f64p)))
        self.next += 1
        return rows[:min(n.value, 64)].copy()

    def launches_per_barrier(self):
        out = C.c_int64()
        check(lib().tgnn_run_launches_per_barrier(self.h, C.byref(out)))
        return out.value

    def close(self):
        if self.h:
            lib().tgnn_run_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def write_dataset(csv_path, num_nodes: int, boundary: int, src, dst, t, efeat=None):
    """write_dataset (temporal_graph.hpp:237-262): CSV + .meta sidecar; efeat f64 [E, d_e]."""
    src = np.ascontiguousarray(src, np.int64)
    dst = np.ascontiguousarray(dst, np.int64)
    t = np.ascontiguousarray(t, np.float64)
    ef = np.zeros((len(t), 0)) if efeat is None else np.ascontiguousarray(efeat, np.float64)
    check(lib().tgnn_write_dataset(os.fsencode(csv_path), num_nodes, boundary, len(t), _p(src, i64p),
                                   _p(dst, i64p), _p(t, f64p), _p(ef, f64p) if ef.size else None,
                                   ef.shape[1] if ef.ndim == 2 else 0))


def chronological_split(num_events: int, train_frac: float, val_frac: float):
    """chronological_split (temporal_graph.hpp:264-279) -> (train_end, val_end)."""
    a, b = C.c_int64(), C.c_int64()
    check(lib().tgnn_chronological_split(num_events, train_frac, val_frac, C.byref(a), C.byref(b)))
    return a.value, b.value


def write_oplog(path_or_file, rows):
    """A memory copy's op-log (OpLogWriter::append, oplog.hpp:31-35) from the
    rows of all its ranks (Run.oplog()), ordered by (iter, kind, rank): each
    pair's read bracket, then its write bracket, ranks ascending."""
    rows = np.asarray(rows, np.int64).reshape(-1, 6)
    order = np.lexsort((rows[:, 3], rows[:, 2], rows[:, 1]))
    text = "".join("%d,%d,%s,%d,%d,%d\n" % (r[0], r[1], "RW"[r[2]], r[3], r[4], r[5]) for r in rows[order])
    if hasattr(path_or_file, "write"):
        path_or_file.write(text)
    else:
        with open(path_or_file, "w") as f:
            f.write(text)


def save_checkpoint(model: ModelConfig, params, path):
    """save_checkpoint (model.hpp:170-186): model.ckpt the reference CLI can load."""
    p = np.ascontiguousarray(params, np.float64)
    if p.size != param_count(model):
        raise ShapeError("save_checkpoint: flat parameter vector has the wrong length")
    check(lib().tgnn_checkpoint_save(C.byref(model.c()), _p(p, f64p), os.fsencode(path)))


def load_checkpoint(model: ModelConfig, path) -> np.ndarray:
    """load_checkpoint (model.hpp:188-222) into the canonical flat f64 vector."""
    out = np.empty(param_count(model), np.float64)
    check(lib().tgnn_checkpoint_load(C.byref(model.c()), os.fsencode(path), _p(out, f64p)))
    return out


def write_metrics_csv(rows, path_or_file):
    """Writes MetricsRow rows with the reference's exact header and number
    formats (write_metrics_header / write_metrics_row, trainer.hpp:607-618)."""
    lines = ["iter,traversed,loss,val_mrr,elapsed_s\n"]
    for r in np.asarray(rows, np.float64).reshape(-1, 5):
        lines.append("%d,%d,%.17g,%.17g,%.3f\n" % (int(r[0]), int(r[1]), r[2], r[3], r[4]))
    text = "".join(lines)
    if hasattr(path_or_file, "write"):
        path_or_file.write(text)
    else:
        with open(path_or_file, "w") as f:
            f.write(text)


class Evaluator:
    """Device evaluate_mrr / replay_batch (trainer.hpp:336-468): forward-only
    workspaces for batches of batch_size events with n_negatives distractors."""

    def __init__(self, ctx: Context, g: "TemporalGraph", model: ModelConfig, batch_size: int,
                 n_negatives: int = 49):
        self.ctx, self.g, self.model = ctx, g, model
        ctx._adopt(self)
        if model.num_nodes == 0:
            model.num_nodes = g.num_nodes
        self.batch_size, self.n_negatives = batch_size, n_negatives
        self.h = C.c_void_p()
        check(lib().tgnn_evaluator_create(ctx.h, g.h, C.byref(model.c()), batch_size, n_negatives,
                                          C.byref(self.h)))

    def evaluate_mrr(self, params, eval_begin: int, eval_end: int, seed: int = 1):
        p = None if params is None else np.ascontiguousarray(params, np.float64)
        mrr, q = C.c_double(), C.c_int64()
        check(lib().tgnn_evaluate_mrr(self.h, None if p is None else _p(p, f64p), eval_begin, eval_end,
                                      seed, C.byref(mrr), C.byref(q)))
        return mrr.value, q.value

    def replay_batch(self, store: "NodeMemoryStore", params, begin: int, end: int):
        p = None if params is None else np.ascontiguousarray(params, np.float64)
        check(lib().tgnn_replay_batch(self.h, store.h, None if p is None else _p(p, f64p), begin, end))

    def candidates(self, begin: int, end: int, seed: int = 1):
        out = np.zeros((end - begin, self.n_negatives), np.int64)
        check(lib().tgnn_eval_candidates(self.h, begin, end, seed, _p(out, i64p)))
        return out

    def close(self):
        if self.h:
            check(lib().tgnn_evaluator_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class RunResult:
    """RunResult, ref trainer.hpp:589-596 (barrier losses + final weights)."""

    barrier_loss: np.ndarray
    params: np.ndarray
    barriers: int = 0
    extra: dict = field(default_factory=dict)


def run_sequential(ctx: Context, g: TemporalGraph, model: ModelConfig, train: TrainConfig,
                   train_begin: int, train_end: int, barriers=None) -> RunResult:
    """run_sequential (trainer.hpp:777-867) at (1,1,1) on one GPU."""
    if train.num_trainers != 1:
        raise ConfigError("run_sequential: requires i = j = k = 1")
    r = Run(ctx, g, model, train, train_begin, train_end)
    n = r.barriers if barriers is None else min(barriers, r.barriers)
    r.step(n)
    res = RunResult(r.losses(0, n), r.params(), r.barriers)
    r.close()
    return res
