"""CPU oracle for the expert-paging MoE hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``xpg`` 0.1.0
(``/root/reference/pkg/src/xpg``).  It is the *checker*: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
``paper_2604_02715_b200`` never imports anything from ``oracle/`` and fails
loudly when its CUDA library is missing.

Pinning: every function below is checked against golden vectors that
``tests/golden/make_golden.py`` dumped from the reference itself (routing
tables, PageTable block traces, ordering logs, per-layer ``layer_forward``
outputs, short ``resident_baseline`` stacks, generator hashes) — see
``tests/test_oracle_golden.py``.  Integer results are bit-exact; float
results agree with the reference to <= 1e-5 relative L2 (BLAS sgemm vs
sgemv summation order is the only difference).
"""

from __future__ import annotations

import numpy as np

U64 = np.uint64
MASK64 = (1 << 64) - 1

# splitmix64 constants (reference pipeline.py:154-159)
_SM_GAMMA = U64(0x9E3779B97F4A7C15)
_SM_MUL1 = U64(0xBF58476D1CE4E5B9)
_SM_MUL2 = U64(0x94D049BB133111EB)

# router mixing constants (reference pipeline.py:166)
_R_SEED = 0x9E37
_R_TOKEN = 0x85EB
_R_LAYER = 0xC2B2

WEIGHT_STD = np.float32(0.02)  # reference model.py:28 / :211


# ---------------------------------------------------------------------------
# integer arithmetic: splitmix64 + hash router


def splitmix64(x):
    """Vectorised splitmix64 over uint64 (reference pipeline.py:154-159)."""
    x = np.asarray(x, dtype=U64)
    with np.errstate(over="ignore"):
        z = x + _SM_GAMMA
        z = (z ^ (z >> U64(30))) * _SM_MUL1
        z = (z ^ (z >> U64(27))) * _SM_MUL2
    return z ^ (z >> U64(31))


def router_keys(seed: int, tokens, layer: int, num_experts: int):
    """uint64 hash inputs [len(tokens), L] for experts j = 1..L.

    The reference evaluates ``seed*0x9E37 + token*0x85EB + layer*0xC2B2 + j``
    in arbitrary precision before the mod-2^64 mask (pipeline.py:155,166),
    which equals uint64 wrap-around arithmetic with seed reduced mod 2^64.
    """
    base = ((int(seed) * _R_SEED) + int(layer) * _R_LAYER) & MASK64
    t = np.asarray(tokens, dtype=U64)
    j = np.arange(1, num_experts + 1, dtype=U64)
    with np.errstate(over="ignore"):
        return U64(base) + t[:, None] * U64(_R_TOKEN) + j[None, :]


def route(seed: int, num_tokens: int, layer: int, num_experts: int, top_k: int) -> np.ndarray:
    """Routed expert ids (1-based, ascending) for tokens 0..T-1 of one layer.

    Restates ``routed_experts`` (reference pipeline.py:162-170): keep the
    min(top_k, L) smallest (score, j) pairs, return them sorted by j.
    Output: int32 [T, min(top_k, L)].
    """
    k = min(top_k, num_experts)
    if num_tokens == 0:
        return np.zeros((0, k), dtype=np.int32)
    scores = splitmix64(router_keys(seed, np.arange(num_tokens), layer, num_experts))
    # stable argsort keeps ascending j among equal scores == (score, j) order
    order = np.argsort(scores, axis=1, kind="stable")[:, :k]
    return np.sort(order + 1, axis=1).astype(np.int32)


def route_all(seed: int, num_tokens: int, num_layers: int, num_experts: int, top_k: int) -> np.ndarray:
    """int32 [N, T, min(k, L)] routing table for layers 1..N."""
    return np.stack(
        [route(seed, num_tokens, layer, num_experts, top_k) for layer in range(1, num_layers + 1)]
    )


# ---------------------------------------------------------------------------
# geometry (reference model.py:54-127, paging.py:29-77)


def sigma(H: int, F: int, kind: int) -> int:
    return 2 * H * 2 * F if kind == 1 else 2 * F * H


def tensor_offset(N: int, L: int, H: int, F: int, layer: int, expert: int, kind: int) -> int:
    s1, s2 = sigma(H, F, 1), sigma(H, F, 2)
    off = (layer - 1) * L * (s1 + s2) + (expert - 1) * (s1 + s2)
    return off + (s1 if kind == 2 else 0)


def target_layer(i: int, n: int) -> int:
    """Layer recycled when materialising layer i (reference paging.py:29-38)."""
    return ((i - 3 + n) % n) + 1


def slot_closed_form(iteration: int, layer: int, expert: int, N: int, L: int) -> int:
    """1-based block id of (iteration, layer, expert) under the reference
    schedule with a host-only / alpha-split placement."""
    g = (iteration - 1) * N + (layer - 1)
    return (g % 2) * L + expert


def simulate_schedule(N: int, L: int, iterations: int):
    """Independent restatement of the sequential StreamedRunner schedule.

    Reference: pipeline.py:335-360 (materialise), :368-384 (forward),
    :412-426 (sequential order), paging.py:148-206 (lowest-free-first pool).
    Returns (blocks, records): blocks[(it, layer, expert, kind)] = block id in
    map order; records = list of (event, it, layer, kind, tgt_it, tgt_layer)
    in log order.
    """
    free = {1: list(range(1, 2 * L + 1)), 2: list(range(1, 2 * L + 1))}
    bound = {}
    blocks = {}
    records = []
    steps = [(it, ly) for it in range(1, iterations + 1) for ly in range(1, N + 1)]

    def mat(it, ly, kind):
        if it > 1 or ly > 2:
            tgt = target_layer(ly, N)
            tgt_it = it if ly > 2 else it - 1
            records.append(("recycle", it, ly, kind, tgt_it, tgt))
            for e in range(1, L + 1):
                free[kind].append(bound.pop((tgt, e, kind)))
        records.append(("load-start", it, ly, kind, None, None))
        for e in range(1, L + 1):
            free[kind].sort()
            b = free[kind].pop(0)
            bound[(ly, e, kind)] = b
            blocks[(it, ly, e, kind)] = b
        records.append(("load-done", it, ly, kind, None, None))

    for kind in (1, 2):
        mat(*steps[0], kind)
    if len(steps) > 1:
        for kind in (1, 2):
            mat(*steps[1], kind)
    for g, (it, ly) in enumerate(steps):
        records.append(("compute-start", it, ly, None, None, None))
        records.append(("compute-done", it, ly, None, None, None))
        if g + 2 < len(steps):
            for kind in (1, 2):
                mat(*steps[g + 2], kind)
    return blocks, records


def validate_ordering(records) -> list:
    """RAW/WAR replay over (t, event, it, layer, kind, tgt_it, tgt_layer)
    tuples (restates reference pipeline.py:119-147)."""
    first = {}
    for t, ev, it, ly, kind, _ti, _tl in records:
        first.setdefault((ev, it, ly, kind), t)
    out = []
    for t, ev, it, ly, kind, ti, tl in records:
        if ev == "compute-start":
            for d in (1, 2):
                at = first.get(("load-done", it, ly, d))
                if at is None or at >= t:
                    out.append(f"RAW: compute-start iter={it} layer={ly} before load-done kind={d}")
        elif ev == "recycle":
            at = first.get(("compute-done", ti, tl, None))
            if at is None or at >= t:
                out.append(f"WAR: recycle of iter={ti} layer={tl} kind={kind} before its compute-done")
    return out


# ---------------------------------------------------------------------------
# bf16 words and the synthetic generator (reference model.py:130-139, 205-214)


def f32_to_bf16(values) -> np.ndarray:
    bits = np.ascontiguousarray(values, dtype=np.float32).view(np.uint32)
    return ((bits + np.uint32(0x7FFF) + ((bits >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)


def bf16_to_f32(words) -> np.ndarray:
    return (np.asarray(words, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def synth_payload(N: int, L: int, H: int, F: int, seed: int) -> np.ndarray:
    """uint16 words of the whole XPGW payload, bit-identical to the reference."""
    count = N * L * (sigma(H, F, 1) + sigma(H, F, 2)) // 2
    rng = np.random.default_rng(seed)
    return f32_to_bf16(rng.standard_normal(count, dtype=np.float32) * WEIGHT_STD)


def initial_activations(H: int, T: int, seed: int) -> np.ndarray:
    """reference pipeline.py:211-213."""
    return np.random.default_rng(seed ^ 0xA5A5A5).standard_normal((T, H), dtype=np.float32)


class WordPool:
    """Read-only view of a payload (uint16 words, container order)."""

    def __init__(self, N, L, H, F, words):
        self.N, self.L, self.H, self.F = N, L, H, F
        self.words = np.asarray(words, dtype=np.uint16).reshape(-1)

    def tensor_words(self, layer, expert, kind):
        off = tensor_offset(self.N, self.L, self.H, self.F, layer, expert, kind) // 2
        n = sigma(self.H, self.F, kind) // 2
        shape = (2 * self.F, self.H) if kind == 1 else (self.H, self.F)
        return self.words[off:off + n].reshape(shape)

    def tensor_f32(self, layer, expert, kind):
        return bf16_to_f32(self.tensor_words(layer, expert, kind))


class SharedPool:
    """Shared (always-on) experts: uint16 words in (layer, shared expert, kind) order.
    No reference counterpart -- our convention (parity unpinned)."""

    def __init__(self, N, S, H, F, words):
        self.N, self.S, self.H, self.F = N, S, H, F
        self.words = np.asarray(words, dtype=np.uint16).reshape(-1)

    def tensor_f32(self, layer, index, kind):
        eb = sigma(self.H, self.F, 1) + sigma(self.H, self.F, 2)
        off = (((layer - 1) * self.S + (index - 1)) * eb + (sigma(self.H, self.F, 1) if kind == 2 else 0)) // 2
        n = sigma(self.H, self.F, kind) // 2
        shape = (2 * self.F, self.H) if kind == 1 else (self.H, self.F)
        return bf16_to_f32(self.words[off:off + n].reshape(shape))


# ---------------------------------------------------------------------------
# SwiGLU expert + MoE layer (reference pipeline.py:180-208, 216-230)


def silu(x):
    return x * (np.float32(1.0) / (np.float32(1.0) + np.exp(-x)))


def expert_rows(gate_up: np.ndarray, down: np.ndarray, xs: np.ndarray) -> np.ndarray:
    """expert_output for a batch of token rows xs [n, H] -> [n, H] (f32)."""
    f = gate_up.shape[0] // 2
    with np.errstate(over="ignore"):
        g = xs @ gate_up[:f].T
        u = xs @ gate_up[f:].T
        return (silu(g) * u) @ down.T


def layer_forward(pool: WordPool, layer: int, acts: np.ndarray, top_k: int, seed: int,
                  shared: "SharedPool | None" = None) -> np.ndarray:
    """One MoE layer: y_t = sum_{j in routed(t), ascending} expert_j(x_t) * f32(1/top_k).

    Vectorised per expert over its tokens; per-token accumulation order is
    the reference's (ascending j, pipeline.py:203-206).  With ``shared``, each
    shared expert's output is then added with weight 1 (our convention).
    """
    acts = np.asarray(acts, dtype=np.float32)
    T = acts.shape[0]
    routes = route(seed, T, layer, pool.L, top_k)
    inv_k = np.float32(1.0 / top_k)
    per_slot = np.zeros((routes.shape[1], T, pool.H), dtype=np.float32)
    for e in np.unique(routes):
        tok, slot = np.nonzero(routes == e)
        gu = pool.tensor_f32(layer, int(e), 1)
        dn = pool.tensor_f32(layer, int(e), 2)
        per_slot[slot, tok] = expert_rows(gu, dn, acts[tok]) * inv_k
    y = np.zeros_like(acts)
    for s in range(routes.shape[1]):
        y += per_slot[s]
    if shared is not None:
        for i in range(1, shared.S + 1):
            y += expert_rows(shared.tensor_f32(layer, i, 1), shared.tensor_f32(layer, i, 2), acts)
    return y


def layer_forward_shard(pool: WordPool, layer: int, acts: np.ndarray, top_k: int, seed: int, num_experts: int,
                        first: int = 0, shared: "SharedPool | None" = None, shared_rows=None) -> np.ndarray:
    """One expert-parallel rank's share of a layer: ``layer_forward`` over the
    ``num_experts``-wide router (pipeline.py:162-170), keeping only the routed experts
    ``first+1 .. first+pool.L`` whose weights ``pool`` holds in shard-local order; the
    other slots add nothing.  ``shared_rows=(r0, n)``: the rows the shared experts apply
    to (this rank's own tokens; our convention).  Summing the shards of a
    layer gives ``layer_forward`` up to f32 addition order."""
    acts = np.asarray(acts, dtype=np.float32)
    T = acts.shape[0]
    routes = route(seed, T, layer, num_experts, top_k)
    inv_k = np.float32(1.0 / top_k)
    per_slot = np.zeros((routes.shape[1], T, pool.H), dtype=np.float32)
    for e in np.unique(routes):
        if not (first < e <= first + pool.L):
            continue
        tok, slot = np.nonzero(routes == e)
        gu = pool.tensor_f32(layer, int(e) - first, 1)
        dn = pool.tensor_f32(layer, int(e) - first, 2)
        per_slot[slot, tok] = expert_rows(gu, dn, acts[tok]) * inv_k
    y = np.zeros_like(acts)
    for s in range(routes.shape[1]):
        y += per_slot[s]
    if shared is not None:
        r0, n = shared_rows if shared_rows is not None else (0, T)
        for i in range(1, shared.S + 1):
            y[r0:r0 + n] += expert_rows(shared.tensor_f32(layer, i, 1), shared.tensor_f32(layer, i, 2),
                                        acts[r0:r0 + n])
    return y


def resident_stack(pool: WordPool, acts: np.ndarray, top_k: int, seed: int, iterations: int = 1,
                   shared: "SharedPool | None" = None):
    """resident_baseline restated: iterations x layers 1..N."""
    a = np.array(acts, dtype=np.float32, copy=True)
    for _ in range(iterations):
        for layer in range(1, pool.N + 1):
            a = layer_forward(pool, layer, a, top_k, seed, shared)
    return a


def rel_l2(got, want) -> float:
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    num = np.linalg.norm(got - want)
    if den == 0.0:
        return 0.0 if num == 0.0 else float("inf")
    return float(num / den)
