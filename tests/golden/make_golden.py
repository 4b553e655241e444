"""Dump golden vectors from the reference ``xpg`` package (run in the dev
container, where /root/reference exists; the outputs are committed).

    python tests/golden/make_golden.py

Writes tests/golden/golden_v1.npz and tests/golden/golden_v1.json.  The GPU
box never runs this script (it has no /root/reference); the tests only read
the committed fixtures.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from xpg import model as M
    from xpg import pipeline as P
    from xpg import storage as S

    arrays = {}
    meta = {"reference": "xpg 0.1.0 @ /root/reference/pkg/src", "cases": {}}

    # 1. splitmix64 known answers (pipeline.py:154-159)
    xs = [0, 1, 0x9E37, (1 << 64) - 1, 0x0123456789ABCDEF, 1 << 63, 12345678901234567890]
    xs += [(7 * 0x9E37 + t * 0x85EB + 0xC2B2 + j) & ((1 << 64) - 1) for t in range(4) for j in range(1, 9)]
    arrays["kat_in"] = np.array(xs, dtype=np.uint64)
    arrays["kat_out"] = np.array([P._splitmix64(x) for x in xs], dtype=np.uint64)

    # 2. routing tables (pipeline.py:162-170)
    route_cases = [
        (7, 64, 4, 8, 2), (7, 32, 2, 128, 8), (7, 16, 2, 256, 8), (-1, 8, 3, 8, 2),
        ((1 << 64) + 7, 8, 2, 8, 2), (12345678901234567890, 16, 4, 8, 2), (0, 4, 2, 1, 2),
        (5, 6, 4, 3, 4), (9, 8, 8, 4, 3), (-(1 << 70) + 3, 5, 2, 16, 5), (7, 256, 1, 8, 2),
        (7, 64, 1, 128, 8), (7, 64, 1, 256, 8), (2, 7, 3, 64, 1),
    ]
    for ci, (seed, T, N, L, k) in enumerate(route_cases):
        tab = np.array(
            [[P.routed_experts(seed, t, layer, L, k) for t in range(T)] for layer in range(1, N + 1)],
            dtype=np.int32,
        )
        arrays[f"route_{ci}"] = tab
        meta["cases"][f"route_{ci}"] = {"seed": str(seed), "T": T, "N": N, "L": L, "k": k}

    # 3. block ids and ordering logs from the sequential StreamedRunner
    slot_cases = [(2, 1), (2, 3), (3, 1), (4, 2), (5, 3), (6, 2), (8, 4), (4, 8), (3, 5)]
    for ci, (N, L) in enumerate(slot_cases):
        spec = M.ModelSpec(N, L, 4, 4)
        container = M.generate_synthetic_model(spec, 1)
        backends = [S.Backend(1, S.BackendKind.HOST_OFFLOAD, 1e9, 1 << 40)]
        plan = S.plan_placement(spec, backends)
        hier = S.StorageHierarchy(container, None, plan, backends)
        trace = []
        runner = P.StreamedRunner(spec, hier, P.ForwardSpec(2, 2, 1), mode="sequential", trace=trace)
        rep = runner.run(3)
        maps = []
        for line in trace:
            f = dict(kv.split("=") for kv in line.split())
            if f["event"] == "map":
                maps.append((int(f["layer"]), int(f["expert"]), int(f["kind"]), int(f["block"])))
        arrays[f"slots_{ci}"] = np.array(maps, dtype=np.int32)
        ev_code = {"recycle": 0, "load-start": 1, "load-done": 2, "compute-start": 3, "compute-done": 4}
        recs = [
            (ev_code[r.event], r.iteration, r.layer, -1 if r.kind is None else r.kind,
             -1 if r.target_iteration is None else r.target_iteration,
             -1 if r.target_layer is None else r.target_layer)
            for r in rep.records
        ]
        arrays[f"order_{ci}"] = np.array(recs, dtype=np.int32)
        meta["cases"][f"slots_{ci}"] = {"N": N, "L": L, "iterations": 3,
                                        "arena_peak_bytes": rep.arena_peak_bytes,
                                        "trace_lines": len(trace)}

    # 4. per-layer layer_forward on fresh N(0,1) inputs (non-degenerate)
    fwd_cases = [
        # (N, L, H, F, wseed, layer, T, k, rseed)
        (4, 8, 256, 512, 7, 1, 1, 2, 7),
        (4, 8, 256, 512, 7, 2, 4, 2, 7),
        (4, 8, 256, 512, 7, 3, 16, 2, 7),
        (4, 8, 256, 512, 7, 4, 64, 2, 7),
        (4, 8, 256, 512, 7, 1, 256, 2, 7),
        (2, 3, 64, 96, 11, 2, 9, 4, 3),     # L < k: cap at L, scale stays 1/k
        (2, 16, 128, 64, 5, 1, 33, 3, 12345678901234567890),
        (2, 32, 64, 128, 3, 2, 40, 8, -5),
    ]
    for ci, (N, L, H, F, wseed, layer, T, k, rseed) in enumerate(fwd_cases):
        spec = M.ModelSpec(N, L, H, F)
        container = M.generate_synthetic_model(spec, wseed)
        x = np.random.default_rng(1000 + ci).standard_normal((T, H), dtype=np.float32)
        fwd = P.ForwardSpec(T, k, rseed)
        y = P.layer_forward(container.tensor_f32, spec, fwd, layer, x)
        arrays[f"fwd_x_{ci}"] = x
        arrays[f"fwd_y_{ci}"] = y
        meta["cases"][f"fwd_{ci}"] = {
            "N": N, "L": L, "H": H, "F": F, "wseed": wseed, "layer": layer, "T": T, "k": k,
            "rseed": str(rseed), "payload_sha256": hashlib.sha256(container.payload).hexdigest(),
        }

    # 5. short resident stacks (resident_baseline, pipeline.py:216-230)
    stack_cases = [
        # (N, L, H, F, wseed, T, k, iterations)
        (4, 8, 256, 512, 7, 16, 2, 1),
        (3, 4, 64, 128, 2, 8, 2, 2),
    ]
    for ci, (N, L, H, F, wseed, T, k, iters) in enumerate(stack_cases):
        spec = M.ModelSpec(N, L, H, F)
        container = M.generate_synthetic_model(spec, wseed)
        fwd = P.ForwardSpec(T, k, wseed)
        x = P.initial_activations(spec, fwd, wseed)
        y = P.resident_baseline(iters, spec, container, fwd, acts=x)
        arrays[f"stack_x_{ci}"] = x
        arrays[f"stack_y_{ci}"] = y
        meta["cases"][f"stack_{ci}"] = {"N": N, "L": L, "H": H, "F": F, "wseed": wseed, "T": T,
                                        "k": k, "iterations": iters,
                                        "payload_sha256": hashlib.sha256(container.payload).hexdigest()}

    # 6. generator hashes (model.py:205-214) and bf16 conversions (model.py:130-139)
    for (N, L, H, F, seed) in [(2, 2, 4, 8, 1), (4, 8, 256, 512, 7), (2, 3, 64, 96, 11)]:
        c = M.generate_synthetic_model(M.ModelSpec(N, L, H, F), seed)
        meta["cases"][f"gen_{N}_{L}_{H}_{F}_{seed}"] = hashlib.sha256(c.payload).hexdigest()
    vals = np.random.default_rng(99).standard_normal(4096, dtype=np.float32) * np.float32(3.0)
    vals[:6] = [1.0, 0.0, -2.0, 0.02, 1.00390625, 1.01171875]  # exact + RNE tie cases
    arrays["bf16_in"] = vals
    arrays["bf16_out"] = M.float32_to_bf16(vals)

    # 7. placement plans (storage.py:92-187): assignment [N][L][2] of backend ids
    import random

    place_cases = []
    rnd = random.Random(7)
    for trial in range(12):
        spec = M.ModelSpec(rnd.randint(2, 4), rnd.randint(1, 6), 8 * rnd.randint(1, 4), 8 * rnd.randint(1, 4))
        nb = rnd.randint(1, 3)
        bws = [rnd.uniform(1e8, 1e10) for _ in range(nb)]
        kinds = [S.BackendKind.HOST_OFFLOAD] * nb
        alpha = None
        if nb == 2 and trial % 2 == 0:
            kinds = [S.BackendKind.COMPRESSED_DEVICE, S.BackendKind.HOST_OFFLOAD]
            alpha = [0.25, 0.5, 0.125, 1.0, 0.375, 0.75][trial % 6]
        backends = [S.Backend(i + 1, kinds[i], bws[i], 1 << 40) for i in range(nb)]
        plan = S.plan_placement(spec, backends, alpha=alpha)
        tab = np.zeros((spec.num_layers, spec.experts_per_layer, 2), dtype=np.int32)
        for tid, bid in plan.assignment.items():
            tab[tid.layer - 1, tid.expert - 1, int(tid.kind) - 1] = bid
        est = S.estimate_load(plan, backends, spec)
        arrays[f"place_{trial}"] = tab
        meta["cases"][f"place_{trial}"] = {
            "spec": [spec.num_layers, spec.experts_per_layer, spec.hidden_dim, spec.intermediate_dim],
            "backends": [[b.backend_id, b.kind.value, b.bandwidth, b.capacity] for b in backends],
            "alpha": alpha, "fractions": {str(k): v for k, v in plan.fractions.items()},
            "tau_load": est.tau_load,
        }

    # 8. exponent codec (codec.py): tables, per-tensor streams, XPGC bytes
    from xpg import codec as X

    for (N, L, H, F, seed) in [(2, 2, 16, 32, 6), (3, 2, 32, 64, 4), (4, 8, 256, 512, 7)]:
        spec = M.ModelSpec(N, L, H, F)
        container = M.generate_synthetic_model(spec, seed)
        cm = X.CompressedModel.from_container(container)
        key = f"xpgc_{N}_{L}_{H}_{F}_{seed}"
        arrays[key + "_lengths"] = np.array(cm.table.code_lengths, dtype=np.uint8)
        arrays[key + "_bits"] = np.array([len(cm.tensors[t].exponent_bitstream) for t in M.iter_tensor_ids(spec)],
                                         dtype=np.int64)
        arrays[key + "_bitcount"] = np.array([cm.tensors[t].exponent_bit_count for t in M.iter_tensor_ids(spec)],
                                             dtype=np.int64)
        meta["cases"][key] = {"sha256": hashlib.sha256(cm.to_bytes()).hexdigest(), "ratio": cm.ratio}
    adv = np.arange(65536, dtype=np.uint16).astype("<u2").tobytes()
    t_adv = X.build_table(X.build_histogram(adv))
    ct_adv = X.compress(adv, t_adv)
    arrays["codec_adv_lengths"] = np.array(t_adv.code_lengths, dtype=np.uint8)
    meta["cases"]["codec_adv"] = {"stream_sha256": hashlib.sha256(ct_adv.exponent_bitstream).hexdigest(),
                                  "bit_count": ct_adv.exponent_bit_count}
    rnd = np.random.default_rng(9).integers(0, 65536, 200_000, dtype=np.uint16).astype("<u2").tobytes()
    t_rnd = X.build_table(X.build_histogram(rnd))
    ct_rnd = X.compress(rnd, t_rnd)
    arrays["codec_rnd_lengths"] = np.array(t_rnd.code_lengths, dtype=np.uint8)
    meta["cases"]["codec_rnd"] = {"stream_sha256": hashlib.sha256(ct_rnd.exponent_bitstream).hexdigest(),
                                  "bit_count": ct_rnd.exponent_bit_count}
    skew = np.zeros(256, dtype=np.int64)
    skew[:40] = [2 ** min(i, 40) for i in range(40)]  # forces the 32-bit length cap
    arrays["codec_skew_counts"] = skew
    arrays["codec_skew_lengths"] = np.array(X.build_table(X.ExponentHistogram(tuple(int(v) for v in skew))).code_lengths,
                                            dtype=np.uint8)

    np.savez_compressed(os.path.join(HERE, "golden_v1.npz"), **arrays)
    with open(os.path.join(HERE, "golden_v1.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
