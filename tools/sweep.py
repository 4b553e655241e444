"""Sweeps for BASELINE configs 3 and 5 (one JSON line per point).

    python tools/sweep.py budget [--config mixtral] [--tokens 256] [--budgets 0.1,0.15,...]
        expert-HBM budget 10-100%: each budget spent by budget.plan_residency (sub-layer ring,
        compressed device tier, pinned experts); fully-resident comparator beside every point
    python tools/sweep.py budget-ring [--config mixtral] [--rings 6,8,12]
        the reference's geometry instead: sub-layer rings below two layers, then pinning
        experts 1..m of every layer (residency tier x > 0), host tier only
    python tools/sweep.py tokens [--config qwen3] [--list 1,4,16,64,256]
        decode batch sweep under the fixed 2-layer-ring budget
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from bench import CONFIGS, SEED, h2d_peak_gbps  # noqa: E402


def timed(torch, fn, steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    rep = fn(steps)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e-3, rep


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("what", choices=["budget", "budget-ring", "tokens"])
    ap.add_argument("--budgets", default="0.1,0.15,0.2,0.25,0.35,0.5,0.65,0.8,1.0")
    ap.add_argument("--config", default=None)
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--list", default="1,4,16,64,256")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--raw", action="store_true")
    ap.add_argument("--budget", type=float, default=0.25, help="tokens: the expert-HBM budget every point plans for")
    ap.add_argument("--depth", type=int, default=None, help="budget: windows in flight on the planned ring (default: the planner picks 1 or 2)")
    ap.add_argument("--window", type=int, default=None, help="budget: experts per ring window")
    ap.add_argument("--b-dec", type=float, default=None, help="budget: the planner's decoder GB/s (model input)")
    ap.add_argument("--device-format", default="auto", choices=["auto", "huffman", "fx4", "mixed"],
                    help="budget: device-tier records (auto: the planner picks by its step model)")
    ap.add_argument("--stage-bufs", type=int, default=None, help="staging buffers per kind (host codec)")
    ap.add_argument("--rings", default="6,8,12", help="sub-layer ring sizes (expert blocks per kind) for budget")
    args = ap.parse_args()
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    cfg = dict(CONFIGS[args.config or ("qwen3" if args.what == "tokens" else "mixtral")])
    if args.tokens:
        cfg["T"] = args.tokens
    N, L, H, F, k = cfg["N"], cfg["L"], cfg["H"], cfg["F"], cfg["k"]
    S, G = cfg.get("S", 0), cfg.get("ep_virtual", 1)
    spec = X.ModelSpec(N, L, H, F)
    cspec, run_kw = spec, {}
    if G > 1:  # one EP rank's slice on this GPU (as bench.py's dsv3 config)
        from paper_2604_02715_b200.expert_parallel import shard_bounds

        first, count = shard_bounds(L, G)[0]
        cspec = X.ModelSpec(N, count, H, F)
        run_kw = {"expert_shard": (first, count), "shared_tokens": (0, cfg["T"])}
    t0 = time.time()
    container = X.generate_fast_model(cspec, SEED, shared_experts=S)
    shared_b = container.shared.total_bytes if container.shared is not None else 0
    budget_base = cspec.total_bytes + shared_b
    backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
    hier = X.StorageHierarchy(container, None, X.plan_placement(cspec, backends), backends)
    if not args.raw:
        hier.compressed = CompressedModel.from_container(container)
    peak = h2d_peak_gbps(torch, 0)
    print(f"setup {time.time() - t0:.1f}s", file=sys.stderr, flush=True)
    if args.what == "budget-ring":
        points = [("ring", int(r)) for r in args.rings.split(",") if r] + [("pinned", p) for p in range(0, L)]
    elif args.what == "budget":
        points = [("plan", float(b)) for b in args.budgets.split(",") if b]
    else:
        points = [("tokens", int(t)) for t in args.list.split(",")]
    resident_tok = {}
    for what, p in points:
        T = int(p) if what == "tokens" else cfg["T"]
        fwd = X.ForwardSpec(T * G, k, SEED)
        x = torch.from_numpy(X.initial_activations(spec, fwd, SEED)).cuda()
        runner = X.StreamedRunner(spec, hier, fwd, host_codec=not args.raw,
                                  pinned=(p if what == "pinned" else None),
                                  ring_experts=(p if what == "ring" else None), stage_buffers=args.stage_bufs,
                                  **run_kw)
        plan = None
        if what in ("plan", "tokens"):
            from paper_2604_02715_b200.budget import fx4_expert_bytes, plan_tiers

            Lc = cspec.experts_per_layer
            ceb = runner.device_tier_bytes(Lc) / (N * Lc) * 1.002
            b = p if what == "plan" else args.budget
            plan = plan_tiers(N, Lc, spec.expert_bytes, ceb, b * budget_base, shared_bytes=shared_b,
                              fx4_ceb=fx4_expert_bytes(spec.hidden_dim, spec.intermediate_dim) * 1.002,
                              units_per_expert=spec.intermediate_dim // 128,
                              device_format=args.device_format,
                              overhead_bytes=runner.ctx.hbm_bytes()["staging"], depth=args.depth, window=args.window,
                              **({"b_dec": args.b_dec * 1e9} if args.b_dec else {}))
            runner.apply_plan(plan)
        runner.run(args.warmup, acts=x)
        secs, rep = timed(torch, lambda s: runner.run(s, acts=x), args.steps)
        hbm = runner.ctx.hbm_bytes()
        row = {"sweep": args.what, "config": args.config or cfg["name"], "T": T,
               "budget": p if what == "plan" else None,
               "pinned_per_layer": (plan.pinned_experts / N if plan else (p if what == "pinned" else 0)),
               "device_tier_per_layer": plan.device_experts / N if plan else 0,
               "device_format": getattr(plan, "device_format", "huffman") if plan else None,
               "fused_decode": bool(getattr(plan, "fused", False)) if plan else False,
               "fx4_per_layer": plan.fx4_experts / N if plan else 0,
               "planned_tok_s": T / plan.est_step_s if plan else None,
               "ring_depth": plan.depth if plan else 2, "stage_buffers": args.stage_bufs or 4,
               "ring_experts": (plan.ring if plan else (p if what == "ring" else 2 * (L - (p if what == "pinned" else 0)))),
               "hbm_fraction": (hbm["ring"] + hbm["device_tier"]) / budget_base,
               "hbm_footprint": (hbm["ring"] + hbm["staging"] + hbm["device_tier"]) / budget_base,
               "tok_s": T * args.steps / secs, "ms_per_step": 1e3 * secs / args.steps,
               "page_in_gbps": rep.h2d_bytes / rep.elapsed_seconds / 1e9 if rep.elapsed_seconds else 0.0,
               "h2d_peak_gbps": peak, "exposed_xfer_pct": 100 * rep.stall_seconds / max(rep.elapsed_seconds, 1e-12),
               "host_codec": not args.raw}
        del runner
        if T not in resident_tok:
            model = X.ResidentModel(spec, container, max_tokens=T * G, **run_kw)
            model.run(1, fwd, x)
            rs, _ = timed(torch, lambda s: model.run(s, fwd, x), args.steps)
            resident_tok[T] = T * args.steps / rs
            del model
        row["resident_tok_s"] = resident_tok[T]
        row["fraction_of_resident"] = row["tok_s"] / resident_tok[T]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
