"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes binding of oracle/_ref/libtgnn_ref.so,
the unmodified reference headers compiled by oracle/Makefile. Loaded only by
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference leg.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libtgnn_ref.so")

i64p = C.POINTER(C.c_int64)
i32p = C.POINTER(C.c_int32)
f64p = C.POINTER(C.c_double)


class ModelCfg(C.Structure):
    _fields_ = [("d_mem", C.c_int64), ("d_time", C.c_int64), ("d_static", C.c_int64),
                ("d_attn", C.c_int64), ("d_hidden", C.c_int64), ("d_e", C.c_int64),
                ("n_neighbors", C.c_int64), ("num_nodes", C.c_int64), ("max_t", C.c_double)]


class TrainCfg(C.Structure):
    _fields_ = [("i", C.c_int32), ("j", C.c_int32), ("k", C.c_int32), ("p", C.c_int32),
                ("q", C.c_int32), ("epochs", C.c_int32), ("local_batch", C.c_int64),
                ("lr_base", C.c_double), ("seed", C.c_uint64), ("local_batch_ref", C.c_int64),
                ("neg_groups", C.c_int64)]


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"oracle library missing: {LIB_PATH} (run `make -C oracle`)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_param_count.restype = C.c_int64
        _lib.ref_sample_recent_neighbors.restype = C.c_int64
        _lib.ref_adam_create.restype = C.c_void_p
        _lib.ref_adam_create.argtypes = [C.c_int64]
        _lib.ref_adam_free.argtypes = [C.c_void_p]
        _lib.ref_graph_free.argtypes = [C.c_void_p]
    return _lib


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a, t):
    return a.ctypes.data_as(t)


def model_cfg(c) -> ModelCfg:
    return ModelCfg(c.d_mem, c.d_time, c.d_static, c.d_attn, c.d_hidden, c.d_e,
                    c.n_neighbors, c.num_nodes, c.max_t)


def train_cfg(i=1, j=1, k=1, p=1, q=None, epochs=1, local_batch=600, lr_base=1e-3, seed=1,
              local_batch_ref=0, neg_groups=0) -> TrainCfg:
    if q is None:
        q = i * j * k // p
    return TrainCfg(i, j, k, p, q, epochs, local_batch, lr_base, seed, local_batch_ref,
                    neg_groups)


class RefGraph:
    """Owns a reference TemporalGraph (finalized)."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle)
        n, b, e, de = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        lib().ref_graph_info(self.h, C.byref(n), C.byref(b), C.byref(e), C.byref(de))
        self.num_nodes, self.boundary, self.num_events, self.d_e = n.value, b.value, e.value, de.value

    def __del__(self):
        try:
            if self.h:
                lib().ref_graph_free(self.h)
        except Exception:
            pass

    @staticmethod
    def synthetic(nodes, events, d_e=0, seed=1, burst_prob=0.2, pref_prob=0.85,
                  prefs_per_src=3, src_frac=0.5, bipartite=True, zipf_s=1.0):
        out = C.c_void_p()
        _check(lib().ref_graph_synthetic(C.c_int64(nodes), C.c_int64(events),
                                         C.c_double(burst_prob), C.c_double(pref_prob),
                                         C.c_int32(prefs_per_src), C.c_double(src_frac),
                                         C.c_int32(1 if bipartite else 0), C.c_int64(d_e),
                                         C.c_double(zipf_s), C.c_uint64(seed), C.byref(out)))
        return RefGraph(out.value)

    @staticmethod
    def from_events(num_nodes, boundary, src, dst, t, efeat=None, d_e=0):
        src = np.ascontiguousarray(src, np.int64)
        dst = np.ascontiguousarray(dst, np.int64)
        t = np.ascontiguousarray(t, np.float64)
        ef = np.ascontiguousarray(efeat if efeat is not None else np.zeros((len(t), d_e)),
                                  np.float64)
        out = C.c_void_p()
        _check(lib().ref_graph_from_events(C.c_int64(num_nodes), C.c_int64(boundary),
                                           C.c_int64(len(t)), _p(src, i64p), _p(dst, i64p),
                                           _p(t, f64p), _p(ef, f64p), C.c_int64(d_e),
                                           C.byref(out)))
        return RefGraph(out.value)

    @staticmethod
    def load_dataset(csv_path):
        out = C.c_void_p()
        _check(lib().ref_load_dataset(os.fsencode(csv_path), C.byref(out)))
        return RefGraph(out.value)

    def write_dataset(self, csv_path):
        _check(lib().ref_write_dataset(self.h, os.fsencode(csv_path)))

    def run_oplog(self, mcfg, tcfg, train_begin, train_end, prefix):
        """run_training with one op-log file per memory copy: <prefix>.<r>.oplog."""
        mc = model_cfg(mcfg)
        _check(lib().ref_run_oplog(self.h, C.byref(mc), C.byref(tcfg), C.c_int64(train_begin),
                                   C.c_int64(train_end), os.fsencode(prefix)))

    def chronological_split(self, train_frac, val_frac):
        a, b = C.c_int64(), C.c_int64()
        _check(lib().ref_chronological_split(self.h, C.c_double(train_frac), C.c_double(val_frac),
                                             C.byref(a), C.byref(b)))
        return a.value, b.value

    def export(self, feats=True):
        E = self.num_events
        src = np.empty(E, np.int64)
        dst = np.empty(E, np.int64)
        t = np.empty(E, np.float64)
        ef = np.empty((E, self.d_e), np.float64) if feats else None
        lib().ref_graph_export(self.h, _p(src, i64p), _p(dst, i64p), _p(t, f64p),
                               _p(ef, f64p) if feats and self.d_e else None)
        return src, dst, t, ef

    def export_feats(self, begin, end):
        ef = np.empty((end - begin, self.d_e), np.float64)
        if self.d_e:
            lib().ref_graph_export_feats(self.h, C.c_int64(begin), C.c_int64(end), _p(ef, f64p))
        return ef

    # -- sampler ------------------------------------------------------------
    def sample_recent_neighbors(self, v, t, n):
        node = np.empty(max(n, 1), np.int64)
        ev = np.empty(max(n, 1), np.int64)
        dt = np.empty(max(n, 1), np.float64)
        c = lib().ref_sample_recent_neighbors(self.h, C.c_int64(v), C.c_double(t), C.c_int64(n),
                                              _p(node, i64p), _p(ev, i64p), _p(dt, f64p))
        return node[:c], ev[:c], dt[:c]

    def sample_negatives(self, batch_index, group, count, seed):
        out = np.empty(count, np.int64)
        _check(lib().ref_sample_negatives(self.h, C.c_int64(batch_index), C.c_int64(group),
                                          C.c_int64(count), C.c_uint64(seed), _p(out, i64p)))
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
        sup = np.empty(R * (n + 1), np.int64)
        U = C.c_int64()
        _check(lib().ref_plan_sub_batch(self.h, C.c_int64(begin), C.c_int64(end),
                                        _p(negatives, i64p), C.c_int64(n), _p(rn, i64p),
                                        _p(rt, f64p), _p(cnt, i64p), _p(nn, i64p), _p(ne, i64p),
                                        _p(nd, f64p), _p(sup, i64p), C.byref(U)))
        return dict(begin=begin, end=end, root_node=rn, root_t=rt, nbr_count=cnt, nbr_node=nn,
                    nbr_event=ne, nbr_dt=nd, supports=sup[:U.value].copy())

    # -- model ----------------------------------------------------------------
    def sub_step(self, mcfg, params, begin, end, negatives, view_mem, view_mail):
        mc = model_cfg(mcfg)
        n = lib().ref_param_count(C.byref(mc))
        U = view_mem.shape[0]
        grads = np.empty(n, np.float64)
        s_hat = np.empty((U, mcfg.d_mem), np.float64)
        loss = C.c_double()
        params = np.ascontiguousarray(params, np.float64)
        negatives = np.ascontiguousarray(negatives, np.int64)
        vm = np.ascontiguousarray(view_mem, np.float64)
        vl = np.ascontiguousarray(view_mail, np.float64)
        _check(lib().ref_sub_step(self.h, C.byref(mc), _p(params, f64p), C.c_int64(begin),
                                  C.c_int64(end), _p(negatives, i64p), _p(vm, f64p),
                                  _p(vl, f64p), C.byref(loss), _p(grads, f64p),
                                  _p(s_hat, f64p)))
        return loss.value, grads, s_hat

    def build_root_writes(self, d_mem, n, begin, end, negatives, view_mem, view_mail, s_hat):
        B = end - begin
        nodes = np.empty(2 * B, np.int64)
        mem = np.empty((2 * B, d_mem), np.float64)
        mail = np.empty((2 * B, 2 * d_mem + 3), np.float64)
        W = C.c_int64()
        negatives = np.ascontiguousarray(negatives, np.int64)
        vm = np.ascontiguousarray(view_mem, np.float64)
        vl = np.ascontiguousarray(view_mail, np.float64)
        sh = np.ascontiguousarray(s_hat, np.float64)
        _check(lib().ref_build_root_writes(self.h, C.c_int64(d_mem), C.c_int64(n),
                                           C.c_int64(begin), C.c_int64(end),
                                           _p(negatives, i64p), _p(vm, f64p), _p(vl, f64p),
                                           _p(sh, f64p), _p(nodes, i64p), _p(mem, f64p),
                                           _p(mail, f64p), C.byref(W)))
        w = W.value
        return nodes[:w].copy(), mem[:w].copy(), mail[:w].copy()

    def replay_batch(self, mcfg, params, state, begin, end):
        """state: dict of numpy arrays (memory, last_update, mail_mem, mail_t, mail_dt,
        mail_event), updated in place."""
        mc = model_cfg(mcfg)
        params = np.ascontiguousarray(params, np.float64)
        _check(lib().ref_replay_batch(self.h, C.byref(mc), _p(params, f64p),
                                      _p(state["memory"], f64p), _p(state["last_update"], f64p),
                                      _p(state["mail_mem"], f64p), _p(state["mail_t"], f64p),
                                      _p(state["mail_dt"], f64p), _p(state["mail_event"], i64p),
                                      C.c_int64(begin), C.c_int64(end)))

    def eval_candidates(self, begin, end, n_neg, seed):
        out = np.zeros((end - begin, n_neg), np.int64)
        _check(lib().ref_eval_candidates(self.h, C.c_int64(begin), C.c_int64(end), C.c_int32(n_neg),
                                         C.c_uint64(seed), _p(out, i64p)))
        return out

    def evaluate_mrr(self, mcfg, params, begin, end, batch, n_neg, seed):
        mc = model_cfg(mcfg)
        params = np.ascontiguousarray(params, np.float64)
        mrr = C.c_double()
        q = C.c_int64()
        _check(lib().ref_evaluate_mrr(self.h, C.byref(mc), _p(params, f64p), C.c_int64(begin),
                                      C.c_int64(end), C.c_int64(batch), C.c_int32(n_neg),
                                      C.c_uint64(seed), C.byref(mrr), C.byref(q)))
        return mrr.value, q.value

    def run(self, mcfg, tcfg, train_begin, train_end, val_begin=0, val_end=0,
            eval_negatives=49, eval_batch=0, sequential=None, want_params=True):
        mc = model_cfg(mcfg)
        if sequential is None:
            sequential = tcfg.i * tcfg.j * tcfg.k == 1
        cap = 1 << 20
        n = lib().ref_param_count(C.byref(mc))
        bl = np.zeros(cap, np.float64)
        params = np.empty(n, np.float64) if want_params else None
        metrics = np.zeros((4096, 5), np.float64)
        nb, nm, el = C.c_int64(), C.c_int64(), C.c_double()
        _check(lib().ref_run(self.h, C.byref(mc), C.byref(tcfg), C.c_int64(train_begin),
                             C.c_int64(train_end), C.c_int64(val_begin), C.c_int64(val_end),
                             C.c_int32(eval_negatives), C.c_int64(eval_batch),
                             C.c_int32(1 if sequential else 0), _p(bl, f64p), C.c_int64(cap),
                             C.byref(nb), _p(params, f64p) if want_params else None,
                             _p(metrics, f64p), C.c_int64(4096), C.byref(nm), C.byref(el)))
        return dict(barrier_loss=bl[:nb.value].copy(), params=params,
                    metrics=metrics[:nm.value].copy(), elapsed_s=el.value, barriers=nb.value)


def run_snapshots(graph, mcfg, tcfg, train_begin, train_end, cap=64):
    """run_training with segment_snapshots: (meta [n x 3] = copy, sweep, segment,
    memory [n, N, d_mem], last_update [n, N]) over every memory copy."""
    mc = model_cfg(mcfg)
    N, d = int(mcfg.num_nodes), int(mcfg.d_mem)
    meta = np.zeros((cap, 3), np.int64)
    mem = np.zeros((cap, N, d))
    lu = np.zeros((cap, N))
    n = C.c_int64()
    _check(lib().ref_run_snapshots(graph.h, C.byref(mc), C.byref(tcfg), C.c_int64(train_begin),
                                   C.c_int64(train_end), C.c_int64(cap), C.byref(n), _p(meta, i64p),
                                   _p(mem, f64p), _p(lu, f64p)))
    assert n.value <= cap, "raise cap"
    return meta[:n.value], mem[:n.value], lu[:n.value]


def validate_oplog(path, i, j):
    """validate_oplog_file (oplog.hpp:105-160) -> (ok, line, message)."""
    line = C.c_int64()
    msg = C.create_string_buffer(512)
    _check(lib().ref_validate_oplog(os.fsencode(path), C.c_int32(i), C.c_int32(j), C.byref(line), msg,
                                    C.c_int64(512)))
    return line.value == 0, line.value, msg.value.decode()


def param_count(mcfg) -> int:
    mc = model_cfg(mcfg)
    return lib().ref_param_count(C.byref(mc))


def save_checkpoint(mcfg, params, path):
    mc = model_cfg(mcfg)
    params = np.ascontiguousarray(params, np.float64)
    _check(lib().ref_save_checkpoint(C.byref(mc), _p(params, f64p), os.fsencode(path)))


def load_checkpoint(mcfg, path) -> np.ndarray:
    mc = model_cfg(mcfg)
    out = np.empty(lib().ref_param_count(C.byref(mc)), np.float64)
    _check(lib().ref_load_checkpoint(C.byref(mc), os.fsencode(path), _p(out, f64p)))
    return out


def init_params(mcfg, seed) -> np.ndarray:
    mc = model_cfg(mcfg)
    out = np.empty(lib().ref_param_count(C.byref(mc)), np.float64)
    _check(lib().ref_init_params(C.byref(mc), C.c_uint64(seed), _p(out, f64p)))
    return out


class RefAdam:
    def __init__(self, n):
        self.h = C.c_void_p(lib().ref_adam_create(n))

    def __del__(self):
        try:
            lib().ref_adam_free(self.h)
        except Exception:
            pass

    def step(self, mcfg, params, grads, lr):
        mc = model_cfg(mcfg)
        grads = np.ascontiguousarray(grads, np.float64)
        _check(lib().ref_adam_step(self.h, C.byref(mc), _p(params, f64p), _p(grads, f64p),
                                   C.c_double(lr)))
        return params


def assignment(tcfg, train_begin, train_end):
    """Per-(rank, barrier) task table from the reference build_assignment."""
    T = tcfg.i * tcfg.j * tcfg.k
    cap = 1 << 16
    shape = (T, cap)
    active = np.zeros(shape, np.int32)
    sub = np.zeros(shape, np.int32)
    batch = np.zeros(shape, np.int64)
    sb = np.zeros(shape, np.int64)
    se = np.zeros(shape, np.int64)
    ng = np.zeros(shape, np.int64)
    pair = np.zeros(shape, np.int64)
    sweep = np.zeros(shape, np.int32)
    at = np.zeros(cap, np.int64)
    tr = np.zeros(cap, np.int64)
    ev = np.zeros(cap, np.int64)
    resets = np.zeros((tcfg.k, cap), np.int64)
    nb, ne = C.c_int64(), C.c_int64()
    _check(lib().ref_assignment(C.byref(tcfg), C.c_int64(train_begin), C.c_int64(train_end),
                                C.byref(nb), C.c_int64(cap), _p(active, i32p), _p(sub, i32p),
                                _p(batch, i64p), _p(sb, i64p), _p(se, i64p), _p(ng, i64p),
                                _p(pair, i64p), _p(sweep, i32p), _p(at, i64p), _p(tr, i64p),
                                _p(ev, i64p), C.byref(ne), _p(resets, i64p)))
    b = nb.value
    return dict(barriers=b, active=active[:, :b].copy(), sub=sub[:, :b].copy(),
                batch=batch[:, :b].copy(), slice_begin=sb[:, :b].copy(),
                slice_end=se[:, :b].copy(), neg_group=ng[:, :b].copy(), pair=pair[:, :b].copy(),
                sweep=sweep[:, :b].copy(), active_trainers=at[:b].copy(),
                traversed_after=tr[:b].copy(), eval_barriers=ev[:ne.value].copy(),
                resets=resets[:, :b].copy())
