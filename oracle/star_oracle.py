"""CPU oracle for the Star Attention two-phase hot path — TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference (`starsim` 0.1.0,
/root/reference/pkg/src/starsim) for the functions on the hot path.  It exists
to CHECK the CUDA product path; it is imported only by tests/, by
__graft_entry__.smoke() and by bench.py's `cpu_baseline` / `--impl reference`
legs.  Nothing in paper_2411_17116_b200/ imports it, and the product path
never falls back to it.

Parity is PINNED: tests/test_oracle.py checks every function below against
golden vectors produced by running the unmodified reference in the build
container (tests/golden/make_golden.py), bit-exact for integer/layout items
and at the reference's own tolerances for floating point.

Each function cites the reference file:line it follows (paths relative to
/root/reference/pkg/src/starsim/).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------
# errors (errors.py:4-17)
# ----------------------------------------------------------------------------


class OracleError(ValueError):
    pass


class OShapeError(OracleError):
    pass


class ODomainError(OracleError):
    pass


class OConfigError(OracleError):
    pass


# ----------------------------------------------------------------------------
# splitmix64 counter PRNG (numerics.py:183-263)
# ----------------------------------------------------------------------------
M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB


def mix64_np(z: np.ndarray) -> np.ndarray:
    """Vectorised bijective finaliser (numerics.py:190-196); uint64 wraps mod 2^64."""
    z = z.astype(np.uint64, copy=True)
    z ^= z >> np.uint64(30)
    z *= np.uint64(MIX1)
    z ^= z >> np.uint64(27)
    z *= np.uint64(MIX2)
    z ^= z >> np.uint64(31)
    return z


def draw_u64(seed: int, first: int, n: int) -> np.ndarray:
    """Draws `first`..`first+n-1` (1-based counter) of stream `seed` (numerics.py:205-224)."""
    ctr = np.arange(first, first + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        state = np.uint64(seed & M64) + ctr * np.uint64(GOLDEN)
        return mix64_np(state)


class OraclePrng:
    """Stateful view over the counter stream (numerics.py:199-252)."""

    def __init__(self, seed: int):
        self.seed = int(seed) & M64
        self.count = 0

    def u64(self) -> int:
        self.count += 1
        return int(draw_u64(self.seed, self.count, 1)[0])

    def unit(self) -> float:
        return (self.u64() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        if n <= 0:
            raise ODomainError("below needs n >= 1")
        return self.u64() % n

    def block(self, n: int) -> np.ndarray:
        z = draw_u64(self.seed, self.count + 1, n)
        self.count += n
        return z

    def permuted(self, items) -> list:
        # Fisher-Yates from the top (numerics.py:231-237)
        xs = list(items)
        i = len(xs) - 1
        while i > 0:
            j = self.below(i + 1)
            xs[i], xs[j] = xs[j], xs[i]
            i -= 1
        return xs

    def floyd_sorted(self, n: int, k: int) -> list[int]:
        # Floyd's distinct sample (numerics.py:239-247)
        if k > n:
            raise ODomainError("sample larger than range")
        got: set[int] = set()
        for j in range(n - k, n):
            t = self.below(j + 1)
            got.add(j if t in got else t)
        return sorted(got)


def uniform_fill(prng: OraclePrng, rows: int, cols: int, scale: float, dtype=np.float32) -> np.ndarray:
    """(2u-1)*scale with u = (z>>11)*2^-53, rounded once to dtype (numerics.py:255-263)."""
    if scale <= 0:
        raise ODomainError("scale must be positive")
    z = prng.block(rows * cols)
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return ((2.0 * u - 1.0) * scale).reshape(rows, cols).astype(dtype)


def counter_fill(seed: int, n: int, scale: float = 1.0) -> np.ndarray:
    """Random-access fp64 values of draws 1..n of `seed` (the GPU kernel's contract)."""
    z = draw_u64(seed, 1, n)
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (2.0 * u - 1.0) * scale


# ----------------------------------------------------------------------------
# rotary embedding, adjacent pairs, fp64 angles (numerics.py:161-180)
# ----------------------------------------------------------------------------


def rope(x: np.ndarray, positions, theta: float = 10000.0) -> np.ndarray:
    rows, d = x.shape
    if d % 2:
        raise OConfigError("rope needs even head_dim")
    pos = np.asarray(positions, dtype=np.float64).reshape(-1)
    if pos.size != rows:
        raise OShapeError("one position per row")
    freq = theta ** (-2.0 * np.arange(d // 2) / d)
    ang = np.outer(pos, freq)
    c, s = np.cos(ang), np.sin(ang)
    ev, od = x[:, 0::2].astype(np.float64), x[:, 1::2].astype(np.float64)
    y = np.empty((rows, d), dtype=np.float64)
    y[:, 0::2] = ev * c - od * s
    y[:, 1::2] = ev * s + od * c
    return y.astype(x.dtype)


# ----------------------------------------------------------------------------
# attention math (attention.py:74-210)
# ----------------------------------------------------------------------------


def causal_keep(lq: int, lk: int, q_offset: int = 0) -> np.ndarray:
    """Row i (absolute index q_offset+i) sees keys j <= q_offset+i (attention.py:74-76)."""
    return np.arange(lk)[None, :] <= (np.arange(lq) + q_offset)[:, None]


def masked_attend(q: np.ndarray, k: np.ndarray, v: np.ndarray, keep):
    """Softmax attention returning (out, lse); masked cells are skipped (attention.py:79-106).

    Scores are formed in the input dtype; lse = max + ln(sum) is carried in fp64.
    Rows with no visible key get out=0, lse=-inf.
    """
    sc = (q @ k.T) * q.dtype.type(1.0 / math.sqrt(q.shape[1]))
    if keep is None:
        mx = sc.max(axis=1)
        p = np.exp(sc - mx[:, None])
        tot = p.sum(axis=1)
        lse = mx.astype(np.float64) + np.log(tot.astype(np.float64))
        return (p / tot[:, None]) @ v, lse
    keep = np.asarray(keep, dtype=bool)
    live = keep.any(axis=1)
    mx = np.where(keep, sc, -np.inf).max(axis=1)
    p = np.zeros_like(sc)
    p[keep] = np.exp((sc - mx[:, None])[keep])
    tot = p.sum(axis=1)
    out = np.zeros((q.shape[0], v.shape[1]), dtype=np.result_type(q, v))
    lse = np.full(q.shape[0], -np.inf)
    if live.any():
        out[live] = (p[live] / tot[live, None]) @ v
        lse[live] = mx[live].astype(np.float64) + np.log(tot[live].astype(np.float64))
    return out, lse


def _check(q, k, v):
    if k.shape[0] != v.shape[0]:
        raise OShapeError("k/v row mismatch")
    if q.shape[1] != k.shape[1]:
        raise OShapeError("q/k width mismatch")


def causal_attention(q, k, v, q_offset: int = 0) -> np.ndarray:
    """attention.py:109-122."""
    _check(q, k, v)
    if q_offset + q.shape[0] > k.shape[0]:
        raise OShapeError("query rows extend past keys")
    keep = causal_keep(q.shape[0], k.shape[0], q_offset)
    if not keep.any(axis=1).all():
        raise ODomainError("query row with no keys")
    return masked_attend(q, k, v, keep)[0]


def causal_attention_lse(q, k, v, q_offset: int = 0):
    """Same as causal_attention but also returns the per-row lse (used for K1 parity)."""
    _check(q, k, v)
    return masked_attend(q, k, v, causal_keep(q.shape[0], k.shape[0], q_offset))


def partial_attention(q, k, v, mask="full", q_offset: int = 0):
    """(locally normalised out, fp64 lse) (attention.py:125-151)."""
    _check(q, k, v)
    if isinstance(mask, str):
        if mask == "full":
            keep = None
        elif mask == "causal":
            keep = causal_keep(q.shape[0], k.shape[0], q_offset)
        else:
            raise OConfigError(f"unknown mask {mask!r}")
    else:
        keep = np.asarray(mask, dtype=bool)
        if keep.shape != (q.shape[0], k.shape[0]):
            raise OShapeError("mask shape")
    if k.shape[0] == 0:
        raise ODomainError("empty key set")
    if keep is not None and not keep.any(axis=1).all():
        raise ODomainError("fully masked row")
    out, lse = masked_attend(q, k, v, keep)
    if not np.isfinite(lse).all():
        raise ODomainError("non-finite lse")
    return out, lse


def merge_partials(outs, lses):
    """Fold partials in the given order: s = logaddexp-reduce, w = exp(lse_h - s) (attention.py:154-173)."""
    if len(outs) == 0:
        raise ODomainError("merge of zero partials")
    if len(outs) == 1:
        return outs[0], np.asarray(lses[0], dtype=np.float64)
    L = np.stack([np.asarray(x, dtype=np.float64) for x in lses])
    O = np.stack(outs)
    s = np.logaddexp.reduce(L, axis=0)
    w = np.exp(L - s[None, :])
    return (w[:, :, None] * O).sum(axis=0).astype(O.dtype), s


def streaming_causal_attention(q, k, v, tile: int, q_offset: int = 0) -> np.ndarray:
    """Key-tiled fold with the merge rule (attention.py:176-210)."""
    if tile < 1:
        raise OConfigError("tile >= 1")
    _check(q, k, v)
    lq, lk = q.shape[0], k.shape[0]
    acc = np.zeros((lq, v.shape[1]), dtype=np.result_type(q, v))
    acc_lse = np.full(lq, -np.inf)
    for t0 in range(0, lk, tile):
        t1 = min(lk, t0 + tile)
        keep = np.arange(t0, t1)[None, :] <= (np.arange(lq) + q_offset)[:, None]
        if not keep.any():
            continue
        o, l = masked_attend(q, k[t0:t1], v[t0:t1], keep)
        s = np.logaddexp(acc_lse, l)
        ok = s > -np.inf
        wa = np.zeros(lq)
        wt = np.zeros(lq)
        wa[ok] = np.exp(acc_lse[ok] - s[ok])
        wt[ok] = np.exp(l[ok] - s[ok])
        acc = wa[:, None] * acc + wt[:, None] * o
        acc_lse = s
    if not np.isfinite(acc_lse).all():
        raise ODomainError("query row with no keys")
    return acc.astype(q.dtype)


# ----------------------------------------------------------------------------
# blocking / anchors (blocking.py:49-236)
# ----------------------------------------------------------------------------
CONTENT_MODES = ("first_block", "none", "previous_block", "random_tokens",
                 "shuffled_first_block", "constant_token")
POSITION_MODES = ("first_block", "previous_block", "random_sampled")


@dataclass(frozen=True)
class Plan:
    L: int
    b: int
    n: int
    H: int
    owner: tuple

    def span(self, i):
        lo = i * self.b
        return lo, min(lo + self.b, self.L)

    def blocks_of(self, h):
        return [i for i, o in enumerate(self.owner) if o == h]


def plan_blocks(L: int, b: int, hosts=None, allow_idle=False) -> Plan:
    """n = ceil(L/b); owner[i] = min(i*H//n, H-1) (blocking.py:49-69)."""
    if L < 1 or b < 1:
        raise OConfigError("L and b must be >= 1")
    n = (L + b - 1) // b
    H = n if hosts is None else hosts
    if H < 1 or (H > n and not allow_idle):
        raise OConfigError("bad host count")
    return Plan(L, b, n, H, tuple(min(i * H // n, H - 1) for i in range(n)))


@dataclass(frozen=True)
class Anchor:
    content_mode: str = "first_block"
    position_mode: str = "first_block"
    anchor_len: int | None = None
    constant_token_id: int = 0
    token_range: int = 256


def augmented_blocks(plan: Plan, tokens, spec: Anchor, prng: OraclePrng | None = None):
    """[(token_ids, position_ids, prefix_len)] per block (blocking.py:182-236)."""
    toks = list(tokens)
    if len(toks) != plan.L:
        raise OConfigError("token count != L")
    a = plan.b if spec.anchor_len is None else spec.anchor_len
    if a > plan.b:
        raise OConfigError("anchor longer than block")
    prng = prng or OraclePrng(0)
    res = []
    for i in range(plan.n):
        lo, hi = plan.span(i)
        own_t, own_p = toks[lo:hi], list(range(lo, hi))
        if i == 0 or spec.content_mode == "none":
            res.append((own_t, own_p, 0))
            continue
        cm = spec.content_mode
        if cm == "first_block":
            at = toks[:a]
        elif cm == "previous_block":
            at = toks[lo - a:lo]
        elif cm == "shuffled_first_block":
            at = prng.permuted(toks[:a])
        elif cm == "random_tokens":
            at = [prng.below(spec.token_range) for _ in range(a)]
        elif cm == "constant_token":
            at = [spec.constant_token_id] * a
        else:
            raise OConfigError(cm)
        pm = spec.position_mode
        if pm == "first_block":
            ap = list(range(a))
        elif pm == "previous_block":
            ap = list(range(lo - a, lo))
        elif pm == "random_sampled":
            ap = prng.floyd_sorted(lo, a)
        else:
            raise OConfigError(pm)
        res.append((list(at) + own_t, ap + own_p, a))
    return res


def star_pairs(L: int, b: int, anchor_len=None) -> int:
    """Phase-1 score pairs = sum_i m_i(m_i+1)/2 (baselines.py:143-152)."""
    a = b if anchor_len is None else anchor_len
    n = (L + b - 1) // b
    tot = 0
    for i in range(n):
        own = min(b, L - i * b)
        m = own if i == 0 else own + a
        tot += m * (m + 1) // 2
    return tot


def star_comm(L, b, d, heads, l_q, n_gen, hosts=None) -> int:
    """(H-1)(l_q+n_gen)(d+1)heads (baselines.py:153-154)."""
    n = (L + b - 1) // b
    H = n if hosts is None else hosts
    return (H - 1) * (l_q + n_gen) * (d + 1) * heads


# ----------------------------------------------------------------------------
# toy model (toy_model.py:37-196)
# ----------------------------------------------------------------------------
RMS_EPS = 1e-6


@dataclass
class ToyModel:
    d_model: int
    heads: int
    layers: int
    vocab: int = 256
    ff_mult: int = 2
    seed: int = 0
    theta: float = 10000.0
    dtype: type = np.float32
    emb: np.ndarray = None
    lw: list = field(default_factory=list)
    final_gain: np.ndarray = None

    @property
    def hd(self):
        return self.d_model // self.heads


def build_toy_model(d_model, heads, layers, vocab=256, ff_mult=2, seed=0, theta=10000.0,
                    dtype=np.float32) -> ToyModel:
    """All weights from one stream in declaration order (toy_model.py:93-113)."""
    m = ToyModel(d_model, heads, layers, vocab, ff_mult, seed & M64, theta, dtype)
    p = OraclePrng(m.seed)
    d, ff = d_model, ff_mult * d_model
    s = 1.0 / np.sqrt(d)
    m.emb = uniform_fill(p, vocab, d, s, dtype)

    def gain():
        return (1.0 + uniform_fill(p, 1, d, 0.1, dtype).reshape(-1)).astype(dtype)

    for _ in range(layers):
        w = {}
        for name, r, c in (("wq", d, d), ("wk", d, d), ("wv", d, d), ("wo", d, d),
                           ("w1", d, ff), ("w2", ff, d)):
            w[name] = uniform_fill(p, r, c, s, dtype)
        w["g_attn"] = gain()
        w["g_ffn"] = gain()
        m.lw.append(w)
    m.final_gain = gain()
    return m


def rms(x, g):
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + RMS_EPS) * g.astype(x.dtype)


def layer_forward(m: ToyModel, w, x, positions, attend):
    """Pre-norm attention + SiLU FFN; attention delegated per head (toy_model.py:141-166)."""
    hd = m.hd
    xn = rms(x, w["g_attn"])
    q, k, v = xn @ w["wq"], xn @ w["wk"], xn @ w["wv"]
    heads_out = []
    for h in range(m.heads):
        c = slice(h * hd, (h + 1) * hd)
        heads_out.append(attend(h, rope(q[:, c], positions, m.theta),
                                rope(k[:, c], positions, m.theta), v[:, c]))
    x = x + np.concatenate(heads_out, axis=1) @ w["wo"]
    z = rms(x, w["g_ffn"]) @ w["w1"]
    return x + (z / (1.0 + np.exp(-z))) @ w["w2"]


def embed(m: ToyModel, tokens):
    ids = list(tokens)
    if not ids or min(ids) < 0 or max(ids) >= m.vocab:
        raise ODomainError("bad token ids")
    return m.emb[ids]


def logits(m: ToyModel, x):
    return rms(x, m.final_gain) @ m.emb.T


def forward_global(m: ToyModel, tokens):
    x = embed(m, tokens)
    pos = range(len(x))
    for w in m.lw:
        x = layer_forward(m, w, x, pos, lambda h, q, k, v: causal_attention(q, k, v))
    return logits(m, x)


# ----------------------------------------------------------------------------
# two-phase protocol (sim.py:108-368)
# ----------------------------------------------------------------------------
ANCHOR_SALT = 0xA17C4B10C4ED5EED
CTX_SALT = 0xC0417E875EED5EED
QRY_SALT = 0x0E5710785EED5EED


@dataclass
class OHost:
    index: int
    # channel c = layer*heads + head -> [K rows x hd], [V rows x hd], positions
    K: list = field(default_factory=list)
    V: list = field(default_factory=list)
    pos: list = field(default_factory=list)
    role: str = "context"


@dataclass
class OSession:
    model: ToyModel
    hosts: list
    q_host: int
    ledger: list
    next_position: int
    last_logits: np.ndarray
    generated: list = field(default_factory=list)


def phase1(m: ToyModel, tokens, plan: Plan, spec: Anchor, prng=None):
    """Encode blocks independently, keep own-row K/V per channel (sim.py:108-175)."""
    prng = prng or OraclePrng(m.seed ^ ANCHOR_SALT)
    blocks = augmented_blocks(plan, tokens, spec, prng)
    per_block = []
    for toks, pos, a in blocks:
        x = embed(m, toks)
        kept = []
        for w in m.lw:
            layer_kept = []

            def att(h, q, k, v, _lk=layer_kept, _a=a):
                _lk.append((k[_a:], v[_a:]))
                return causal_attention(q, k, v)

            x = layer_forward(m, w, x, pos, att)
            kept.append(layer_kept)
        per_block.append((kept, pos[a:]))
    hosts = []
    for h in range(plan.H):
        host = OHost(h)
        mine = plan.blocks_of(h)
        for li in range(m.layers):
            for hh in range(m.heads):
                if mine:
                    host.K.append(np.concatenate([per_block[bi][0][li][hh][0] for bi in mine]))
                    host.V.append(np.concatenate([per_block[bi][0][li][hh][1] for bi in mine]))
                    host.pos.append(sum((list(per_block[bi][1]) for bi in mine), []))
                else:
                    host.K.append(np.zeros((0, m.hd), m.dtype))
                    host.V.append(np.zeros((0, m.hd), m.dtype))
                    host.pos.append([])
        hosts.append(host)
    return hosts


def gather_merge(hosts, q_host: int, ch: int, q, own_tail: int, ledger):
    """Per-host partials in ascending host order, then merge (sim.py:178-213)."""
    if own_tail not in (0, q.shape[0]):
        raise OShapeError("own_tail must be 0 or l_q")
    outs, lses = [], []
    for host in hosts:
        K, V = host.K[ch], host.V[ch]
        if K.shape[0] == 0:
            continue
        if host.index == q_host and own_tail:
            keep = np.ones((q.shape[0], K.shape[0]), dtype=bool)
            keep[:, K.shape[0] - own_tail:] = causal_keep(q.shape[0], own_tail)
            o, l = partial_attention(q, K, V, keep)
        else:
            o, l = partial_attention(q, K, V, "full")
        outs.append(o)
        lses.append(l)
        if host.index != q_host and ledger is not None:
            ledger.append((2, host.index, q_host, "partial_out", q.shape[0] * V.shape[1]))
            ledger.append((2, host.index, q_host, "partial_lse", q.shape[0]))
    if not outs:
        raise OConfigError("all caches empty")
    return merge_partials(outs, lses)[0]


def phase2_forward(m: ToyModel, hosts, q_host, tokens, positions, own_tail, ledger):
    """Append-then-attend on the query host, gather/merge per channel (sim.py:254-281)."""
    x = embed(m, tokens)
    qh = hosts[q_host]
    pos = list(positions)
    for li, w in enumerate(m.lw):

        def att(h, q, k, v, _li=li):
            ch = _li * m.heads + h
            qh.K[ch] = np.concatenate([qh.K[ch], k])
            qh.V[ch] = np.concatenate([qh.V[ch], v])
            qh.pos[ch] = qh.pos[ch] + pos
            return gather_merge(hosts, q_host, ch, q, own_tail, ledger)

        x = layer_forward(m, w, x, pos, att)
    return logits(m, x)


def start_session(m: ToyModel, tokens, plan: Plan, spec: Anchor, prng=None, q_host=None):
    """Phase 1 on tokens[:L], query encode under phase 2 (sim.py:284-324)."""
    L = plan.L
    query = list(tokens[L:])
    if not query:
        raise OConfigError("empty query")
    hosts = phase1(m, tokens[:L], plan, spec, prng)
    q_host = len(hosts) - 1 if q_host is None else q_host
    hosts[q_host].role = "query"
    ledger = [(2, q_host, h.index, "query_broadcast", len(query)) for h in hosts if h.index != q_host]
    lg = phase2_forward(m, hosts, q_host, query, range(L, L + len(query)), len(query), ledger)
    return lg, OSession(m, hosts, q_host, ledger, L + len(query), lg[-1])


def decode(sess: OSession, n_tokens: int):
    """Greedy argmax (ties -> lowest id), one phase-2 step per token (sim.py:340-368)."""
    new = []
    for _ in range(n_tokens):
        t = int(np.argmax(sess.last_logits))
        new.append(t)
        sess.generated.append(t)
        for h in sess.hosts:
            if h.index != sess.q_host:
                sess.ledger.append((2, sess.q_host, h.index, "query_broadcast", 1))
        lg = phase2_forward(sess.model, sess.hosts, sess.q_host, [t], [sess.next_position], 0,
                            sess.ledger)
        sess.last_logits = lg[-1]
        sess.next_position += 1
    return new


def ledger_csv(ledger) -> str:
    rows = ["phase,src,dst,kind,scalar_count"] + [f"{a},{b},{c},{d},{e}" for a, b, c, d, e in ledger]
    return "\n".join(rows) + "\n"


def experiment_tokens(seed: int, L: int, l_q: int, vocab: int = 256):
    """Seeded context/query tokens exactly as the CLI draws them (cli.py:145-167)."""
    pc = OraclePrng(seed ^ CTX_SALT)
    pq = OraclePrng(seed ^ QRY_SALT)
    return [pc.below(vocab) for _ in range(L)], [pq.below(vocab) for _ in range(l_q)]
