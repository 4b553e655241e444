"""Time the fully-resident decode step (no per-launch events) -- A/B helper.

    python tools/resident_time.py [--config mixtral] [--tokens 256] [--steps 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"mixtral": (8, 8, 4096, 14336, 2), "qwen3": (8, 128, 2048, 768, 8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--tokens", type=int, default=256)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    import torch

    import paper_2604_02715_b200 as X

    N, L, H, F, k = SHAPES[args.config]
    spec = X.ModelSpec(N, L, H, F)
    fwd = X.ForwardSpec(args.tokens, k, 7)
    container = X.generate_fast_model(spec, 7)
    model = X.ResidentModel(spec, container, max_tokens=args.tokens)
    x = torch.from_numpy(X.initial_activations(spec, fwd, 7)).cuda()
    model.run(3, fwd, x)
    torch.cuda.synchronize()
    out = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        model.run(args.steps, fwd, x)
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / args.steps)
    print(json.dumps({"config": args.config, "tokens": args.tokens, "ms_per_step": out,
                      "pdl": os.environ.get("XPGB_PDL", "1")}))


if __name__ == "__main__":
    main()
