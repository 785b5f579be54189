"""ORACLE / TEST INFRASTRUCTURE ONLY — never imported by the product path.

A float64 numpy restatement of the DistTGL reference hot path
(/root/reference/proj/include/tgnn, "ref" below). Only tests/,
``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may import it;
it is the checker the CUDA path is compared with, never the thing measured.

Parity status: PINNED. tests/test_oracle_golden.py checks every function
here against golden vectors produced by the unmodified reference compiled
in-process (oracle/_ref/libtgnn_ref.so, generator tests/golden/make_golden.py)
and against the reference's own known-answer tests
(ref/tests/test_temporal_graph.cpp:40-70, test_memory_store.cpp:53-139).

Each function cites the reference lines it restates.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15


# ----------------------------------------------------------------- rng.hpp
def splitmix64(x):
    """rng.hpp:12-17 (vectorised over uint64 arrays)."""
    with np.errstate(over="ignore"):
        x = np.asarray(x, dtype=np.uint64) + np.uint64(GAMMA)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return x ^ (x >> np.uint64(31))


def hash64(*args):
    """rng.hpp:19-24: hash64(a) = splitmix64(a); hash64(a, b, rest...) folds left."""
    with np.errstate(over="ignore"):
        a = np.asarray(args[0], dtype=np.uint64)
        if len(args) == 1:
            return splitmix64(a)
        b = np.asarray(args[1], dtype=np.uint64)
        mixed = a ^ (b + np.uint64(GAMMA) + (a << np.uint64(6)) + (a >> np.uint64(2)))
        return hash64(splitmix64(mixed), *args[2:])


class Rng:
    """rng.hpp:28-56 (scalar, Python ints)."""

    def __init__(self, seed: int):
        self.state = int(splitmix64(np.uint64((int(seed) ^ 0xA02BDBF7BB3C0A7) & M64)))

    def next_u64(self) -> int:
        self.state = int(splitmix64(np.uint64(self.state)))
        return self.state

    def next_unit(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def next_below(self, n: int) -> int:
        return self.next_u64() % n

    def next_range(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.next_unit()

    def next_normal(self) -> float:
        u1 = self.next_unit()
        u2 = self.next_unit()
        if u1 < 1e-300:
            u1 = 1e-300
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586 * u2)


def rng_first_u64(seeds):
    """Vectorised first draw of Rng(seed): splitmix64(splitmix64(seed ^ K))."""
    s = np.asarray(seeds, dtype=np.uint64) ^ np.uint64(0xA02BDBF7BB3C0A7)
    return splitmix64(splitmix64(s))


# ----------------------------------------------------------------- graph
@dataclass
class Graph:
    """TemporalGraph after finalize (temporal_graph.hpp:33-95): events in
    ascending (t, file order); per-node ascending incidence (the T-CSR)."""

    num_nodes: int
    boundary: int
    src: np.ndarray
    dst: np.ndarray
    t: np.ndarray
    efeat: np.ndarray  # [E, d_e]
    inc_ptr: np.ndarray = field(default=None)
    inc_eid: np.ndarray = field(default=None)

    @property
    def d_e(self) -> int:
        return self.efeat.shape[1]

    @property
    def num_events(self) -> int:
        return len(self.t)

    def incident(self, v):
        return self.inc_eid[self.inc_ptr[v]:self.inc_ptr[v + 1]]


def finalize(num_nodes, boundary, src, dst, t, efeat):
    """temporal_graph.hpp:55-91: stable sort by t, validate, build incidence."""
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    t = np.asarray(t, np.float64)
    efeat = np.asarray(efeat, np.float64).reshape(len(t), -1)
    if num_nodes <= 0:
        raise ValueError("graph: num_nodes must be positive")
    if boundary >= 0 and (boundary <= 0 or boundary >= num_nodes):
        raise ValueError("graph: bipartite boundary leaves an empty partition")
    order = np.argsort(t, kind="stable")
    src, dst, t, efeat = src[order], dst[order], t[order], efeat[order]
    if np.any((src < 0) | (src >= num_nodes) | (dst < 0) | (dst >= num_nodes)):
        raise ValueError("graph: node id out of range")
    if boundary >= 0 and np.any(~((src < boundary) & (dst >= boundary))):
        raise ValueError("graph: event does not cross the bipartite boundary")
    E = len(t)
    # each event listed under src then dst; ascending event id per node
    nodes = np.empty(2 * E, np.int64)
    nodes[0::2] = src
    nodes[1::2] = dst
    eids = np.repeat(np.arange(E, dtype=np.int64), 2)
    o = np.argsort(nodes, kind="stable")
    inc_eid = eids[o]
    counts = np.bincount(nodes, minlength=num_nodes)
    inc_ptr = np.zeros(num_nodes + 1, np.int64)
    inc_ptr[1:] = np.cumsum(counts)
    return Graph(num_nodes, boundary, src, dst, t, efeat, inc_ptr, inc_eid)


def sample_recent_neighbors(g: Graph, v: int, t: float, n: int):
    """temporal_graph.hpp:296-318: up to n most recent events of v strictly
    before t, most recent first. Returns (nodes, events, dts)."""
    inc = g.incident(v)
    have = int(np.searchsorted(g.t[inc], t, side="left"))
    take = min(n, have)
    ev = inc[have - take:have][::-1]
    other = np.where(g.src[ev] == v, g.dst[ev], g.src[ev])
    return other.astype(np.int64), ev.astype(np.int64), (t - g.t[ev]).astype(np.float64)


def sample_negatives(g: Graph, batch_index: int, group: int, count: int, seed: int):
    """temporal_graph.hpp:355-370."""
    lo = g.boundary if g.boundary >= 0 else 0
    span = g.num_nodes - lo
    if span <= 0:
        raise ValueError("negative sampling: empty destination partition")
    i = np.arange(count, dtype=np.uint64)
    h = hash64(np.uint64(seed), np.uint64(0x6E656761), np.uint64(batch_index & M64),
               np.uint64(group & M64), i)
    return (lo + (rng_first_u64(h) % np.uint64(span)).astype(np.int64)).astype(np.int64)


def eval_candidates(g: Graph, begin: int, end: int, n_neg: int, seed: int):
    """evaluate_mrr distractors (trainer.hpp:413-423): candidate s of event e is
    lo + Rng(hash64(seed, "eval", e, s)).next_below(span), redrawn while it
    equals the event's destination."""
    lo = g.boundary if g.boundary >= 0 else 0
    span = g.num_nodes - lo
    out = np.zeros((end - begin, n_neg), np.int64)
    for e in range(begin, end):
        dst = int(g.dst[e])
        for s in range(n_neg):
            r = Rng(int(hash64(np.uint64(seed), np.uint64(0x6576616C), np.uint64(e), np.uint64(s))))
            v = lo + r.next_below(span)
            while v == dst:
                v = lo + r.next_below(span)
            out[e - begin, s] = v
    return out


@dataclass
class Plan:
    """SubBatchPlan (trainer.hpp:47-56) in padded array form."""

    begin: int
    end: int
    root_node: np.ndarray   # [R]
    root_t: np.ndarray      # [R]
    nbr_count: np.ndarray   # [R]
    nbr_node: np.ndarray    # [R, n] (-1 padded)
    nbr_event: np.ndarray   # [R, n]
    nbr_dt: np.ndarray      # [R, n]
    supports: np.ndarray    # [U] ascending


def plan_sub_batch(g: Graph, begin: int, end: int, negatives, n: int) -> Plan:
    """trainer.hpp:76-106: roots event-major (src, dst, neg); supports are the
    sorted unique union of roots and their neighbours."""
    B = end - begin
    negatives = np.asarray(negatives, np.int64)
    if len(negatives) != B:
        raise ValueError("plan_sub_batch: one negative per event required")
    R = 3 * B
    root_node = np.empty(R, np.int64)
    root_node[0::3] = g.src[begin:end]
    root_node[1::3] = g.dst[begin:end]
    root_node[2::3] = negatives
    root_t = np.repeat(g.t[begin:end], 3)
    nbr_count = np.zeros(R, np.int64)
    nbr_node = np.full((R, n), -1, np.int64)
    nbr_event = np.full((R, n), -1, np.int64)
    nbr_dt = np.zeros((R, n), np.float64)
    for r in range(R):
        nn, ne, nd = sample_recent_neighbors(g, int(root_node[r]), float(root_t[r]), n)
        c = len(nn)
        nbr_count[r] = c
        nbr_node[r, :c] = nn
        nbr_event[r, :c] = ne
        nbr_dt[r, :c] = nd
    allnodes = np.concatenate([root_node, nbr_node[nbr_node >= 0]])
    return Plan(begin, end, root_node, root_t, nbr_count, nbr_node, nbr_event, nbr_dt,
                np.unique(allnodes))


# ----------------------------------------------------------------- model
@dataclass
class ModelConfig:
    """model.hpp:19-35."""

    d_mem: int = 100
    d_time: int = 100
    d_static: int = 100
    d_attn: int = 100
    d_hidden: int = 0
    d_e: int = 0
    n_neighbors: int = 10
    num_nodes: int = 0
    max_t: float = 1.0

    @property
    def mail_dim(self):
        return 2 * self.d_mem + self.d_time + self.d_e

    @property
    def node_dim(self):
        return self.d_mem + self.d_static

    @property
    def q_in_dim(self):
        return self.node_dim + self.d_time

    @property
    def kv_in_dim(self):
        return self.node_dim + self.d_e + self.d_time

    @property
    def hidden_dim(self):
        return self.d_hidden if self.d_hidden else self.d_mem


TENSOR_ORDER = ["omega", "gru.Wz", "gru.Wr", "gru.Wh", "gru.bz", "gru.br", "gru.bh",
                "attn.Wq", "attn.bq", "attn.Wk", "attn.bk", "attn.Wv", "attn.bv",
                "static_table", "dec.W1", "dec.b1", "dec.W2", "dec.b2"]


def tensor_shapes(c: ModelConfig):
    """shape_params, model.hpp:78-99, in for_each_tensor order (model.hpp:56-76)."""
    gin = c.mail_dim + c.d_mem
    return [
        ("omega", (c.d_time,)),
        ("gru.Wz", (c.d_mem, gin)), ("gru.Wr", (c.d_mem, gin)), ("gru.Wh", (c.d_mem, gin)),
        ("gru.bz", (c.d_mem,)), ("gru.br", (c.d_mem,)), ("gru.bh", (c.d_mem,)),
        ("attn.Wq", (c.d_attn, c.q_in_dim)), ("attn.bq", (c.d_attn,)),
        ("attn.Wk", (c.d_attn, c.kv_in_dim)), ("attn.bk", (c.d_attn,)),
        ("attn.Wv", (c.d_attn, c.kv_in_dim)), ("attn.bv", (c.d_attn,)),
        ("static_table", (c.num_nodes, c.d_static)),
        ("dec.W1", (c.hidden_dim, 2 * c.d_attn)), ("dec.b1", (c.hidden_dim,)),
        ("dec.W2", (1, c.hidden_dim)), ("dec.b2", (1,)),
    ]


def param_count(c: ModelConfig) -> int:
    return sum(int(np.prod(s)) for _, s in tensor_shapes(c))


def unflatten(c: ModelConfig, flat):
    out, at = {}, 0
    for name, shape in tensor_shapes(c):
        k = int(np.prod(shape))
        out[name] = np.asarray(flat[at:at + k], np.float64).reshape(shape)
        at += k
    return out


def flatten(c: ModelConfig, tensors) -> np.ndarray:
    return np.concatenate([np.asarray(tensors[name], np.float64).reshape(-1)
                           for name, _ in tensor_shapes(c)])


def init_params(c: ModelConfig, seed: int) -> np.ndarray:
    """model.hpp:122-141: rank-2 tensors except omega/static get U(+-1/sqrt(cols))
    from Rng(hash64(seed, 'init', slot)); biases/static zero; omega log-spaced."""
    tensors = {}
    for slot, (name, shape) in enumerate(tensor_shapes(c), start=1):
        t = np.zeros(shape, np.float64)
        if not (name in ("omega", "static_table", "dec.b2") or len(shape) < 2):
            seed_h = int(hash64(np.uint64(seed), np.uint64(0x696E6974), np.uint64(slot)))
            rng = Rng(seed_h)
            bound = 1.0 / math.sqrt(float(shape[1]))
            flat = t.reshape(-1)
            for x in range(flat.size):
                flat[x] = rng.next_range(-bound, bound)
        tensors[name] = t
    dt = c.d_time
    for i in range(dt):
        frac = 1.0 if dt == 1 else i / (dt - 1)
        tensors["omega"][i] = math.pow(10.0, -5.0 * (1.0 - frac)) / max(c.max_t, 1e-12)
    return flatten(c, tensors)


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-x))


def softplus(x):
    """decoder.hpp:79-81."""
    return np.maximum(x, 0.0) + np.log1p(np.exp(-np.abs(x)))


# ----------------------------------------------------------------- memory
@dataclass
class MemoryState:
    """NodeMemoryState, memory_store.hpp:16-50."""

    memory: np.ndarray
    last_update: np.ndarray
    mail_mem: np.ndarray
    mail_t: np.ndarray
    mail_dt: np.ndarray
    mail_event: np.ndarray

    @staticmethod
    def init(num_nodes, d_mem):
        return MemoryState(np.zeros((num_nodes, d_mem)), np.zeros(num_nodes),
                           np.zeros((num_nodes, 2 * d_mem)), np.zeros(num_nodes),
                           np.zeros(num_nodes), np.full(num_nodes, -1, np.int64))

    def copy(self):
        return MemoryState(*(a.copy() for a in (self.memory, self.last_update, self.mail_mem,
                                                self.mail_t, self.mail_dt, self.mail_event)))

    def read(self, nodes):
        """DirectMemoryClient::read (shared_buffers.hpp:138-153) + pack_mail_row
        (memory_store.hpp:73-80): mem [U, d], mail [U, 2d+3]."""
        nodes = np.asarray(nodes, np.int64)
        mail = np.concatenate([self.mail_mem[nodes], self.mail_t[nodes, None],
                               self.mail_dt[nodes, None],
                               self.mail_event[nodes, None].astype(np.float64)], axis=1)
        return self.memory[nodes].copy(), mail

    def write(self, nodes, mem_rows, mail_rows):
        """DirectMemoryClient::write -> apply_root_write (memory_store.hpp:168-181),
        rows applied in order so later rows win."""
        d = self.memory.shape[1]
        for x, v in enumerate(np.asarray(nodes, np.int64)):
            self.memory[v] = mem_rows[x]
            self.mail_mem[v] = mail_rows[x, :2 * d]
            self.mail_t[v] = mail_rows[x, 2 * d]
            self.mail_dt[v] = mail_rows[x, 2 * d + 1]
            self.mail_event[v] = int(mail_rows[x, 2 * d + 2])
            self.last_update[v] = mail_rows[x, 2 * d]

    def reset(self):
        """reset_state, memory_store.hpp:43-50."""
        for a in (self.memory, self.last_update, self.mail_mem, self.mail_t, self.mail_dt):
            a[...] = 0.0
        self.mail_event[...] = -1


def comb(nodes, events, ts):
    """memory_store.hpp:121-136: per node keep max (t, event); ascending node.
    Returns the kept indices into the candidate arrays."""
    best = {}
    for x, (v, e, t) in enumerate(zip(nodes, events, ts)):
        b = best.get(int(v))
        if b is None or t > ts[b] or (t == ts[b] and e > events[b]):
            best[int(v)] = x
    return np.array([best[v] for v in sorted(best)], np.int64)


# ----------------------------------------------------------------- step
def _slices(c: ModelConfig):
    d, ds, de, dt = c.d_mem, c.d_static, c.d_e, c.d_time
    return d, ds, de, dt


def freshen(c: ModelConfig, P, g: Graph, mem, mail):
    """freshen_memory (trainer.hpp:111-124) + make_mail (model.hpp:153-166) +
    gru_update (gru.hpp:32-67), vectorised over rows. Returns s_hat and the tape."""
    d = c.d_mem
    ev = mail[:, 2 * d + 2].astype(np.int64)
    has = ev >= 0
    dts = mail[:, 2 * d + 1]
    U = mem.shape[0]
    s_hat = mem.copy()
    phi = np.cos(dts[:, None] * P["omega"][None, :])
    ef = g.efeat[np.where(has, ev, 0)] if c.d_e else np.zeros((U, 0))
    m = np.concatenate([mail[:, :2 * d], phi, ef], axis=1)
    ms = np.concatenate([m, mem], axis=1)
    z = sigmoid(ms @ P["gru.Wz"].T + P["gru.bz"])
    r = sigmoid(ms @ P["gru.Wr"].T + P["gru.br"])
    mrs = np.concatenate([m, r * mem], axis=1)
    h = np.tanh(mrs @ P["gru.Wh"].T + P["gru.bh"])
    new = (1.0 - z) * mem + z * h
    s_hat[has] = new[has]
    return s_hat, dict(has=has, dts=dts, ms=ms, mrs=mrs, z=z, r=r, h=h, s=mem)


def sub_step(c: ModelConfig, flat_params, g: Graph, plan: Plan, view_mem, view_mail):
    """sub_step, trainer.hpp:170-272 (forward + analytic backward; gradients in
    canonical flat order). Returns (loss, grads_flat, s_hat)."""
    P = unflatten(c, flat_params)
    G = {k: np.zeros_like(v) for k, v in P.items()}
    d, ds, de, dtm = _slices(c)
    sup = plan.supports
    row_of = {int(v): i for i, v in enumerate(sup)}
    s_hat, tape = freshen(c, P, g, view_mem, view_mail)

    R = len(plan.root_node)
    ones = np.cos(0.0 * P["omega"])
    q_in = np.concatenate([s_hat[[row_of[int(v)] for v in plan.root_node]],
                           P["static_table"][plan.root_node],
                           np.broadcast_to(ones, (R, dtm))], axis=1)
    q = q_in @ P["attn.Wq"].T + P["attn.bq"]
    h = np.zeros((R, c.d_attn))
    kv_rows, Ks, Vs, As = [], [], [], []
    for r in range(R):
        n = int(plan.nbr_count[r])
        if n == 0:
            kv_rows.append(None); Ks.append(None); Vs.append(None); As.append(None)
            continue
        w = plan.nbr_node[r, :n]
        kv = np.concatenate([s_hat[[row_of[int(x)] for x in w]], P["static_table"][w],
                             g.efeat[plan.nbr_event[r, :n]] if de else np.zeros((n, 0)),
                             np.cos(plan.nbr_dt[r, :n, None] * P["omega"][None, :])], axis=1)
        K = kv @ P["attn.Wk"].T + P["attn.bk"]
        V = kv @ P["attn.Wv"].T + P["attn.bv"]
        sc = (K @ q[r]) / math.sqrt(n)
        a = np.exp(sc - sc.max())
        a /= a.sum()
        h[r] = a @ V
        kv_rows.append(kv); Ks.append(K); Vs.append(V); As.append(a)

    W1, b1, W2, b2 = P["dec.W1"], P["dec.b1"], P["dec.W2"], P["dec.b2"]
    hs, hd, hn = h[0::3], h[1::3], h[2::3]
    in_pos = np.concatenate([hs, hd], axis=1)
    in_neg = np.concatenate([hs, hn], axis=1)
    hid_pos = np.maximum(in_pos @ W1.T + b1, 0.0)
    hid_neg = np.maximum(in_neg @ W1.T + b1, 0.0)
    pos = hid_pos @ W2[0] + b2[0]
    neg = hid_neg @ W2[0] + b2[0]
    ne = len(pos)
    loss = softplus(-pos).sum() / ne + softplus(neg).sum() / ne  # bce_loss decoder.hpp:85-98
    dpos = -sigmoid(-pos) / ne
    dneg = sigmoid(neg) / ne

    # decode_link_backward (decoder.hpp:55-77)
    dh = np.zeros_like(h)
    for dl, hid, inp, other in ((dpos, hid_pos, in_pos, 1), (dneg, hid_neg, in_neg, 2)):
        G["dec.b2"][0] += dl.sum()
        G["dec.W2"][0] += dl @ hid
        dhid = np.where(hid > 0, dl[:, None] * W2[0][None, :], 0.0)
        G["dec.W1"] += dhid.T @ inp
        G["dec.b1"] += dhid.sum(0)
        din = dhid @ W1
        dh[0::3] += din[:, :c.d_attn]
        dh[other::3] += din[:, c.d_attn:]

    # attention_backward + routing (attention.hpp:96-140, trainer.hpp:228-257)
    ds_hat = np.zeros_like(s_hat)
    Wq, Wk, Wv = P["attn.Wq"], P["attn.Wk"], P["attn.Wv"]
    for r in range(R):
        n = int(plan.nbr_count[r])
        if n == 0:
            continue
        a, K, V, kv = As[r], Ks[r], Vs[r], kv_rows[r]
        scale = 1.0 / math.sqrt(n)
        dV = a[:, None] * dh[r][None, :]
        G["attn.Wv"] += dV.T @ kv
        G["attn.bv"] += dV.sum(0)
        da = V @ dh[r]
        dz = a * (da - (a * da).sum())
        gsc = dz * scale
        dq = gsc @ K
        dK = gsc[:, None] * q[r][None, :]
        G["attn.Wk"] += dK.T @ kv
        G["attn.bk"] += dK.sum(0)
        dkv = dV @ Wv + dK @ Wk
        G["attn.Wq"] += np.outer(dq, q_in[r])
        G["attn.bq"] += dq
        dq_in = dq @ Wq
        u = row_of[int(plan.root_node[r])]
        ds_hat[u] += dq_in[:d]
        if ds:
            G["static_table"][plan.root_node[r]] += dq_in[d:d + ds]
        # time slice at dt = 0 contributes -0*sin(0) = 0 to omega
        w = plan.nbr_node[r, :n]
        for m_ in range(n):
            wu = row_of[int(w[m_])]
            ds_hat[wu] += dkv[m_, :d]
            if ds:
                G["static_table"][w[m_]] += dkv[m_, d:d + ds]
            dtv = plan.nbr_dt[r, m_]
            G["omega"] += dkv[m_, d + ds + de:] * (-dtv * np.sin(dtv * P["omega"]))

    # gru_backward (gru.hpp:71-112) + omega at the mail dt (trainer.hpp:259-269)
    has = tape["has"]
    if has.any():
        z, rr, hh, s = tape["z"][has], tape["r"][has], tape["h"][has], tape["s"][has]
        ms, mrs, dts = tape["ms"][has], tape["mrs"][has], tape["dts"][has]
        dsn = ds_hat[has]
        md = c.mail_dim
        da_z = dsn * (hh - s) * z * (1.0 - z)
        da_h = dsn * z * (1.0 - hh * hh)
        G["gru.Wh"] += da_h.T @ mrs
        G["gru.bh"] += da_h.sum(0)
        d_mrs = da_h @ P["gru.Wh"]
        da_r = d_mrs[:, md:] * s * rr * (1.0 - rr)
        G["gru.Wz"] += da_z.T @ ms
        G["gru.bz"] += da_z.sum(0)
        G["gru.Wr"] += da_r.T @ ms
        G["gru.br"] += da_r.sum(0)
        d_ms = da_z @ P["gru.Wz"] + da_r @ P["gru.Wr"]
        dm = d_ms[:, :md] + d_mrs[:, :md]
        dphi = dm[:, 2 * d:2 * d + dtm]
        G["omega"] += (dphi * (-dts[:, None] * np.sin(dts[:, None] * P["omega"][None, :]))).sum(0)

    return float(loss), flatten(c, G), s_hat


def build_root_writes(c: ModelConfig, g: Graph, plan: Plan, view_mem, view_mail, s_hat):
    """trainer.hpp:284-330: two mails per event from the STALE view, dt from the
    cached mail time (0 when none), COMB, rows ascending by node.
    Returns (nodes, mem_rows [W, d], mail_rows [W, 2d+3])."""
    d = c.d_mem
    row_of = {int(v): i for i, v in enumerate(plan.supports)}
    cn, ce, ct, cdt, cm = [], [], [], [], []
    for e in range(plan.begin, plan.end):
        for self_, other in ((g.src[e], g.dst[e]), (g.dst[e], g.src[e])):
            u, o = row_of[int(self_)], row_of[int(other)]
            has = view_mail[u, 2 * d + 2] >= 0
            t_minus = view_mail[u, 2 * d] if has else 0.0
            cn.append(int(self_)); ce.append(e); ct.append(g.t[e]); cdt.append(g.t[e] - t_minus)
            cm.append(np.concatenate([view_mem[u], view_mem[o]]))
    kept = comb(cn, ce, ct)
    nodes = np.array([cn[x] for x in kept], np.int64)
    mem_rows = np.stack([s_hat[row_of[int(v)]] for v in nodes]) if len(nodes) else np.zeros((0, d))
    mail_rows = np.stack([np.concatenate([cm[x], [ct[x], cdt[x], float(ce[x])]]) for x in kept]) \
        if len(kept) else np.zeros((0, 2 * d + 3))
    return nodes, mem_rows, mail_rows


def replay_batch(c: ModelConfig, flat_params, g: Graph, state: MemoryState, begin, end):
    """trainer.hpp:336-371 (+ generate_mails memory_store.hpp:93-119)."""
    if begin >= end:
        return
    P = unflatten(c, flat_params)
    roots = np.unique(np.concatenate([g.src[begin:end], g.dst[begin:end]]))
    mem, mail = state.read(roots)
    s_hat, _ = freshen(c, P, g, mem, mail)
    d = c.d_mem
    cn, ce, ct, cdt, cm = [], [], [], [], []
    for e in range(begin, end):
        for self_, other in ((g.src[e], g.dst[e]), (g.dst[e], g.src[e])):
            cn.append(int(self_)); ce.append(e); ct.append(g.t[e])
            cdt.append(g.t[e] - state.last_update[self_])
            cm.append(np.concatenate([state.memory[self_], state.memory[other]]))
    kept = comb(cn, ce, ct)
    ridx = {int(v): i for i, v in enumerate(roots)}
    rows_mem = np.stack([s_hat[ridx[cn[x]]] for x in kept])
    rows_mail = np.stack([np.concatenate([cm[x], [ct[x], cdt[x], float(ce[x])]]) for x in kept])
    state.write([cn[x] for x in kept], rows_mem, rows_mail)


def embed_roots(c: ModelConfig, P, g: Graph, root_node, root_t, nodes, s_hat):
    """embed_root (trainer.hpp:128-159) + attention_forward (attention.hpp:36-91)
    for each (node, t) root against the freshened support rows s_hat[nodes]."""
    row_of = {int(v): i for i, v in enumerate(nodes)}
    de, dtm = c.d_e, c.d_time
    ones = np.cos(0.0 * P["omega"])
    h = np.zeros((len(root_node), c.d_attn))
    for r, (v, t) in enumerate(zip(root_node, root_t)):
        q_in = np.concatenate([s_hat[row_of[int(v)]], P["static_table"][int(v)], ones])
        q = P["attn.Wq"] @ q_in + P["attn.bq"]
        w, ev, dts = sample_recent_neighbors(g, int(v), float(t), c.n_neighbors)
        n = len(w)
        if n == 0:
            continue
        kv = np.concatenate([s_hat[[row_of[int(x)] for x in w]], P["static_table"][w],
                             g.efeat[ev] if de else np.zeros((n, 0)),
                             np.cos(dts[:, None] * P["omega"][None, :])], axis=1)
        K = kv @ P["attn.Wk"].T + P["attn.bk"]
        V = kv @ P["attn.Wv"].T + P["attn.bv"]
        sc = (K @ q) / math.sqrt(n)
        a = np.exp(sc - sc.max())
        a /= a.sum()
        h[r] = a @ V
    return h


def evaluate_mrr(c: ModelConfig, flat_params, g: Graph, eval_begin, eval_end, batch, n_neg, seed):
    """evaluate_mrr (trainer.hpp:383-468): memory rebuilt by replaying
    [0, eval_begin); each event ranks its destination against n_neg
    distractors, ties counting against it. Returns (mrr, queries)."""
    P = unflatten(c, flat_params)
    state = MemoryState.init(g.num_nodes, c.d_mem)
    for b in range(0, eval_begin, batch):
        replay_batch(c, flat_params, g, state, b, min(eval_begin, b + batch))
    W1, b1, W2, b2 = P["dec.W1"], P["dec.b1"], P["dec.W2"], P["dec.b2"]

    def decode(hu, hv):
        return float(np.maximum(W1 @ np.concatenate([hu, hv]) + b1, 0.0) @ W2[0] + b2[0])

    acc, queries = 0.0, 0
    for b in range(eval_begin, eval_end, batch):
        e_end = min(eval_end, b + batch)
        cand = eval_candidates(g, b, e_end, n_neg, seed)
        root_node, root_t = [], []
        for e in range(b, e_end):
            for v in [g.src[e], g.dst[e], *cand[e - b]]:
                root_node.append(int(v))
                root_t.append(float(g.t[e]))
        nodes = set(root_node)
        for v, t in zip(root_node, root_t):
            nodes.update(int(x) for x in sample_recent_neighbors(g, v, t, c.n_neighbors)[0])
        nodes = np.array(sorted(nodes), np.int64)
        mem, mail = state.read(nodes)
        s_hat, _ = freshen(c, P, g, mem, mail)
        h = embed_roots(c, P, g, root_node, root_t, nodes, s_hat)
        per = 2 + n_neg
        for x in range(e_end - b):
            base = x * per
            truth = decode(h[base], h[base + 1])
            worse = sum(1 for s_ in range(n_neg) if decode(h[base], h[base + 2 + s_]) >= truth)
            acc += 1.0 / (1 + worse)
            queries += 1
        replay_batch(c, flat_params, g, state, b, e_end)
    return (acc / queries if queries else 0.0), queries


class Adam:
    """optimizer.hpp:33-61 (dense, beta=(0.9, 0.999), eps=1e-8)."""

    def __init__(self, n):
        self.m = np.zeros(n)
        self.v = np.zeros(n)
        self.t = 0

    def step(self, params, grads, lr):
        self.t += 1
        c1 = 1.0 - math.pow(0.9, self.t)
        c2 = 1.0 - math.pow(0.999, self.t)
        self.m = 0.9 * self.m + (1.0 - 0.9) * grads
        self.v = 0.999 * self.v + (1.0 - 0.999) * grads * grads
        params -= lr * (self.m / c1) / (np.sqrt(self.v / c2) + 1e-8)
        return params


def lr_eff(lr_base, i, j, k, local_batch, local_batch_ref=0):
    """TrainConfig::lr_eff, parallel.hpp:30-34."""
    ref = local_batch_ref if local_batch_ref > 0 else local_batch
    return lr_base * (i * j * k * local_batch) / ref


def run_sequential(c: ModelConfig, g: Graph, seed: int, local_batch: int, lr_base: float,
                   train_begin: int, train_end: int, epochs: int = 1, barriers=None):
    """run_sequential at (1,1,1) (trainer.hpp:777-867): per barrier plan, read,
    sub_step, write, Adam; memory resets at each sweep start. Returns
    (barrier losses, final params)."""
    params = init_params(c, seed)
    adam = Adam(len(params))
    state = MemoryState.init(g.num_nodes, c.d_mem)
    nb = (train_end - train_begin + local_batch - 1) // local_batch
    total = nb * epochs
    if barriers is not None:
        total = min(total, barriers)
    losses = []
    for b in range(total):
        batch = b % nb
        if batch == 0:
            state.reset()
        lo = train_begin + batch * local_batch
        hi = min(train_end, lo + local_batch)
        negs = sample_negatives(g, batch, b, hi - lo, seed)
        plan = plan_sub_batch(g, lo, hi, negs, c.n_neighbors)
        vm, vl = state.read(plan.supports)
        loss, grads, s_hat = sub_step(c, params, g, plan, vm, vl)
        nodes, mrow, lrow = build_root_writes(c, g, plan, vm, vl, s_hat)
        state.write(nodes, mrow, lrow)
        params = adam.step(params, grads, lr_eff(lr_base, 1, 1, 1, local_batch))
        losses.append(loss)
    return np.array(losses), params
