"""Resident single-layer MoE forward for ncu captures and per-kernel timing.

    python tools/profile_layer.py [--config mixtral] [--tokens 256] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"mixtral": (2, 8, 4096, 14336, 2), "qwen3": (2, 128, 2048, 768, 8), "dsv3": (2, 32, 7168, 2048, 8),
          "tiny": (2, 8, 256, 512, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--sweep", default="")
    args = ap.parse_args()
    import torch

    import paper_2604_02715_b200 as X

    N, L, H, F, k = SHAPES[args.config]
    spec = X.ModelSpec(N, L, H, F)
    t0 = time.time()
    c = X.generate_fast_model(spec, 7)
    model = X.ResidentModel(spec, c, max_tokens=max([args.tokens] + [int(t) for t in args.sweep.split(",") if t]))
    print(f"setup {time.time() - t0:.1f}s", file=sys.stderr)
    toks = [int(t) for t in args.sweep.split(",") if t] or [args.tokens]
    for T in toks:
        x = torch.randn(T, H, device="cuda")
        y = torch.empty_like(x)
        model.ctx.layer_forward(1, x, y, T, k, 7)
        torch.cuda.synchronize()
        prof = model.ctx.profile_layer(1, x, y, T, k, 7, reps=args.reps)
        gu = prof["gate_up_bytes"] / prof["gate_up_ns"]
        dn = prof["down_bytes"] / prof["down_ns"]
        print(json.dumps({"config": args.config, "T": T, **prof, "gate_up_GBps": gu, "down_GBps": dn}))


if __name__ == "__main__":
    main()
