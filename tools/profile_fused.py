"""Decode-into-GEMM vs decode-into-ring on one device-tier-only paged stack.

    python tools/profile_fused.py [--config mixtral] [--layers 2] [--tokens 256] [--steps 5]

Every expert sits compressed on the device tier (alpha = 1); a 2-layer ring.  Prints one JSON
line per mode: ms per decode step, raw-equivalent GB/s of expert weights consumed per step,
and the per-launch gate/up and down kernel times the runner's profile events measured.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"mixtral": (8, 4096, 14336, 2), "qwen3": (128, 2048, 768, 8), "dsv3": (32, 7168, 2048, 8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--modes", default="1,0")
    ap.add_argument("--no-profile", action="store_true", help="no per-launch events (they serialise the launches)")
    ap.add_argument("--act-planes", type=int, default=2, choices=[1, 2])
    ap.add_argument("--device-format", default="huffman", choices=["huffman", "fx4"])
    args = ap.parse_args()
    import numpy as np
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    L, H, F, k = SHAPES[args.config]
    spec = X.ModelSpec(args.layers, L, H, F)
    fwd = X.ForwardSpec(args.tokens, k, 7)
    container = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(spec, backends, alpha=1.0), backends)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((args.tokens, H), dtype=np.float32)).cuda()
    outs = {}
    for mode in (int(m) for m in args.modes.split(",")):
        runner = X.StreamedRunner(spec, hier, fwd, fused_decode=bool(mode), device_format=args.device_format)
        runner.ctx.set_activation_planes(args.act_planes)
        runner.run(1, acts=x.clone())
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep = runner.run(args.steps, acts=x.clone(), profile=not args.no_profile)
        e1.record()
        torch.cuda.synchronize()
        assert rep.page_fault is None and rep.violations == []
        ms = e0.elapsed_time(e1) / args.steps
        outs[mode] = rep.final_activations.cpu().numpy().tobytes()
        print(json.dumps({"config": args.config, "layers": args.layers, "T": args.tokens, "fused": mode,
                          "device_format": args.device_format, "device_tier_bytes": runner.ctx.hbm_bytes()["device_tier"],
                          "ms_per_step": ms, "raw_GBps": spec.total_bytes / ms / 1e6,
                          "tok_s": args.tokens / ms * 1e3, "decoded_bytes_per_step": rep.decoded_bytes / args.steps,
                          "kernels": rep.kernels}), flush=True)
        del runner
        torch.cuda.empty_cache()
    if len(outs) == 2:
        print(json.dumps({"bit_identical": len(set(outs.values())) == 1}))


if __name__ == "__main__":
    main()
