"""CPU restatement of the reference's streamed decode path, for timing — TEST/BENCH
INFRASTRUCTURE ONLY (bench.py ``cpu_baseline`` and ``--impl reference`` legs).

Follows the host-only, sequential reference schedule step for one layer:

* page-in: every expert tensor of the layer is copied from the container
  payload into an arena block (StorageHierarchy.fetch host branch,
  storage.py:235-243, into PageTable.loading_view, paging.py:217-226);
* forward: per token row t, per routed expert j (ascending): copy the page
  out of the arena (read_page, paging.py:228-237), widen bf16 -> f32
  (pipeline.py:364-366), SwiGLU with float32 numpy matvecs (expert_output,
  pipeline.py:184-189), accumulate ``y += out * f32(1/top_k)``
  (pipeline.py:198-207).

The reference runs exactly this work per layer; the timing of one layer on a
few tokens is the bounded sample the bench extrapolates from.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import xpg_oracle as O


def _silu(x):
    return x * (np.float32(1.0) / (np.float32(1.0) + np.exp(-x)))


def streamed_layer(words: np.ndarray, N: int, L: int, H: int, F: int, layer: int, acts: np.ndarray,
                   top_k: int, seed: int):
    """Returns (y, fetch_seconds, compute_seconds)."""
    s1, s2 = O.sigma(H, F, 1) // 2, O.sigma(H, F, 2) // 2
    t0 = time.perf_counter()
    arena = np.empty(L * (s1 + s2), dtype=np.uint16)
    for e in range(1, L + 1):
        off1 = O.tensor_offset(N, L, H, F, layer, e, 1) // 2
        off2 = O.tensor_offset(N, L, H, F, layer, e, 2) // 2
        arena[(e - 1) * s1:e * s1] = words[off1:off1 + s1]
        arena[L * s1 + (e - 1) * s2:L * s1 + e * s2] = words[off2:off2 + s2]
    t1 = time.perf_counter()
    routes = O.route(seed, acts.shape[0], layer, L, top_k)
    inv_k = np.float32(1.0 / top_k)
    out = np.zeros_like(acts)
    with np.errstate(over="ignore"):
        for t in range(acts.shape[0]):
            x = acts[t]
            y = np.zeros_like(x)
            for j in routes[t]:
                j = int(j)
                gu = O.bf16_to_f32(arena[(j - 1) * s1:j * s1].copy()).reshape(2 * F, H)
                dn = O.bf16_to_f32(arena[L * s1 + (j - 1) * s2:L * s1 + j * s2].copy()).reshape(H, F)
                g = gu[:F] @ x
                u = gu[F:] @ x
                y += (dn @ (_silu(g) * u)) * inv_k
            out[t] = y
    t2 = time.perf_counter()
    return out, t1 - t0, t2 - t1


def decode_rate(words: np.ndarray, N: int, L: int, H: int, F: int, T: int, top_k: int, seed: int,
                sample_tokens: int, layer: int = 1):
    """Time one layer on `sample_tokens` rows; extrapolate the reference's per-step
    cost N * (fetch + T * per_token) to decode tokens/s at batch T."""
    x = np.random.default_rng(seed).standard_normal((sample_tokens, H), dtype=np.float32)
    _, t_fetch, t_comp = streamed_layer(words, N, L, H, F, layer, x, top_k, seed)
    per_token = t_comp / max(sample_tokens, 1)
    step = N * (t_fetch + T * per_token)
    return {
        "tok_s": T / step,
        "fetch_s": t_fetch,
        "compute_s": t_comp,
        "per_token_s": per_token,
        "step_s": step,
        "threads": int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1)),
    }


def decode_rate_sampled(tensor_words, N: int, L: int, H: int, F: int, T: int, top_k: int, seed: int,
                        sample_tokens: int, layer: int = 1, shared_words=None):
    """decode_rate for models too large to hold a layer on the host: the page-in of the
    experts the sample routes to is timed and scaled to all L experts of the layer.
    tensor_words(layer, expert, kind) -> uint16 words; shared_words(kind) -> the layer's
    shared expert (added with weight 1, our convention) or None."""
    x = np.random.default_rng(seed).standard_normal((sample_tokens, H), dtype=np.float32)
    routes = O.route(seed, sample_tokens, layer, L, top_k)
    need = sorted({int(j) for j in routes.reshape(-1)})
    s1, s2 = O.sigma(H, F, 1) // 2, O.sigma(H, F, 2) // 2
    t0 = time.perf_counter()
    arena = {}
    for j in need:
        arena[j] = (np.array(tensor_words(layer, j, 1), copy=True), np.array(tensor_words(layer, j, 2), copy=True))
    t1 = time.perf_counter()
    inv_k = np.float32(1.0 / top_k)
    with np.errstate(over="ignore"):
        for t in range(sample_tokens):
            y = np.zeros(H, dtype=np.float32)
            for j in routes[t]:
                gu = O.bf16_to_f32(arena[int(j)][0].copy()).reshape(2 * F, H)
                dn = O.bf16_to_f32(arena[int(j)][1].copy()).reshape(H, F)
                y += (dn @ (_silu(gu[:F] @ x[t]) * (gu[F:] @ x[t]))) * inv_k
            if shared_words is not None:
                gu = O.bf16_to_f32(np.asarray(shared_words(1))).reshape(2 * F, H)
                dn = O.bf16_to_f32(np.asarray(shared_words(2))).reshape(H, F)
                y += dn @ (_silu(gu[:F] @ x[t]) * (gu[F:] @ x[t]))
    t2 = time.perf_counter()
    t_fetch = (t1 - t0) * L / max(1, len(need))
    per_token = (t2 - t1) / max(sample_tokens, 1)
    step = N * (t_fetch + T * per_token)
    return {"tok_s": T / step, "fetch_s": t_fetch, "compute_s": t2 - t1, "per_token_s": per_token, "step_s": step,
            "threads": int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1)),
            "fetched_experts": len(need)}
