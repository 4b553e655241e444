"""Operator commands for the B200 paged MoE path.

    python -m paper_2604_02715_b200 generate OUT.xpgw [--model N,L,H,F] [--seed S]
    python -m paper_2604_02715_b200 compress IN.xpgw OUT.xpgc
    python -m paper_2604_02715_b200 verify IN.xpgw IN.xpgc
    python -m paper_2604_02715_b200 run [--model ...] [--tokens T --top-k K --iterations I] [--alpha A]
                                        [--mode threaded|sequential] [--host-codec] [--container IN.xpgw]
    python -m paper_2604_02715_b200 calibrate [--model ...] [--tokens T --top-k K]

``run`` is the reference's parity run (xpg cli.py:92-165) on the GPU: the streamed
pipeline against the resident baseline, bit-identical output plus a clean
ordering log, same summary fields.  ``calibrate`` measures what the reference's
simulator takes as inputs (simulate.py:20-72) on this GPU -- host-tier and
device-tier bandwidth, per-iteration compute -- and prints them with the
closed-form knee alpha* (simulate.py:156-164).

Exit codes follow the reference (cli.py:24-27): 0 ok, 1 validation error,
2 correctness failure, 3 I/O or runtime error.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

EXIT_OK, EXIT_VALIDATION, EXIT_CORRECTNESS, EXIT_IO = 0, 1, 2, 3


def _spec(args):
    from .geometry import ModelSpec

    n, l, h, f = (int(v) for v in args.model.split(","))
    return ModelSpec(n, l, h, f)


def _model_args(p):
    p.add_argument("--model", default="8,8,64,128", help="N,L,H,F (layers, experts, hidden, ffn)")
    p.add_argument("--seed", type=int, default=7)


def cmd_generate(args) -> int:
    from .errors import ConfigError
    from .geometry import generate_synthetic_model

    if Path(args.out).exists() and not args.force:
        raise ConfigError(f"{args.out} exists; pass --force to overwrite")
    c = generate_synthetic_model(_spec(args), args.seed, pin=False)
    c.write(args.out)
    print(f"wrote {args.out}: {c.spec.total_bytes} payload bytes (seed={args.seed})")
    return EXIT_OK


def cmd_compress(args) -> int:
    from .errors import ConfigError
    from .exponent_codec import CompressedModel
    from .geometry import open_container

    if Path(args.out).exists() and not args.force:
        raise ConfigError(f"{args.out} exists; pass --force to overwrite")
    c = open_container(args.infile, register=False)
    cm = CompressedModel.from_container(c, pin=False)
    cm.write(args.out)
    print(f"wrote {args.out}: payload ratio {cm.ratio:.4f}")
    return EXIT_OK


def cmd_verify(args) -> int:
    from .exponent_codec import CompressedModel
    from .geometry import iter_tensor_ids, open_container

    c = open_container(args.infile, register=False)
    cm = CompressedModel.read(args.compressed)
    for tid in iter_tensor_ids(c.spec):
        if c.tensor_bytes(tid) != cm.tensor_bytes(tid):
            print(f"MISMATCH at {tid}", file=sys.stderr)
            return EXIT_CORRECTNESS
    print(f"identical; payload ratio {cm.ratio:.4f}")
    return EXIT_OK


def _hierarchy(spec, container, alpha):
    from .tiers import Backend, BackendKind, StorageHierarchy, plan_placement

    if alpha is None:
        backends = [Backend(1, BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
    else:
        backends = [Backend(1, BackendKind.COMPRESSED_DEVICE, 500e9, 1 << 50),
                    Backend(2, BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
    return StorageHierarchy(container, None, plan_placement(spec, backends, alpha=alpha), backends)


def cmd_run(args) -> int:
    from .geometry import generate_synthetic_model, initial_activations, open_container
    from .streamed import ForwardSpec, StreamedRunner, resident_baseline

    results, worst = [], EXIT_OK
    for k in range(args.seeds):
        seed = args.seed + k
        container = open_container(args.container) if args.container else generate_synthetic_model(_spec(args), seed)
        spec = container.spec
        fwd = ForwardSpec(args.tokens, args.top_k, seed)
        acts = initial_activations(spec, fwd, seed)
        runner = StreamedRunner(spec, _hierarchy(spec, container, args.alpha), fwd, mode=args.mode,
                                host_codec=args.host_codec)
        rep = runner.run(args.iterations, acts=acts.copy())
        base = resident_baseline(args.iterations, spec, container, fwd, acts=acts.copy())
        identical = rep.page_fault is None and rep.final_activations.tobytes() == base.tobytes()
        results.append({
            "seed": seed, "bit_identical": identical, "violations": len(rep.violations),
            "page_fault": rep.page_fault, "arena_peak_bytes": rep.arena_peak_bytes,
            "expected_peak_bytes": 2 * spec.experts_per_layer * spec.expert_bytes,
            "stall_ms": rep.stall_seconds * 1e3, "checksum": rep.checksum,
            "h2d_bytes": rep.h2d_bytes, "page_in_gbps": rep.page_in_gbps,
        })
        if not identical or rep.violations:
            worst = EXIT_CORRECTNESS
    doc = {"runs": results, "passed": worst == EXIT_OK}
    text = json.dumps(doc, indent=2)
    if args.out:
        Path(args.out).write_text(text)
    print(text)
    return worst


def cmd_calibrate(args) -> int:
    import torch

    from .geometry import generate_fast_model, initial_activations
    from .residency import calibrate_bandwidths, measured_taus
    from .streamed import ForwardSpec, ResidentModel, StreamedRunner

    spec = _spec(args)
    container = generate_fast_model(spec, args.seed)
    fwd = ForwardSpec(args.tokens, args.top_k, args.seed)
    x = torch.from_numpy(initial_activations(spec, fwd, args.seed)).cuda()
    runner = StreamedRunner(spec, _hierarchy(spec, container, None), fwd, host_codec=True)
    b_dev, b_host = calibrate_bandwidths(runner, x)
    rep = runner.run(2, acts=x)
    tau_comp, tau_load = measured_taus(rep)
    # the decoder inside the pipeline: every expert on the device tier, decoded into the ring
    # on the SMs the GEMMs also use (raw bytes per second of the SM time left after compute)
    runner.set_device_experts([spec.experts_per_layer] * spec.num_layers)
    runner.run(1, acts=x)
    rep_dev = runner.run(3, acts=x)
    # the FX4 device tier read in place by the decode-into-GEMM kernel (GEMM included)
    runner.set_device_format("fx4", fused_decode=True)
    runner.run(1, acts=x)
    rep_fx4 = runner.run(3, acts=x)
    runner.set_device_format("huffman", fused_decode=False)
    runner.set_device_experts([0] * spec.num_layers)
    del runner
    model = ResidentModel(spec, container, max_tokens=args.tokens)
    model.run(1, fwd, x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    model.run(3, fwd, x)
    e1.record()
    torch.cuda.synchronize()
    tau_resident = e0.elapsed_time(e1) * 1e-3 / 3
    sm_time = rep_dev.elapsed_seconds / 3 - tau_resident
    b_dec_pipeline = spec.total_bytes / sm_time if sm_time > 0 else float("inf")
    b_fx4_fused = 3 * spec.total_bytes / rep_fx4.elapsed_seconds if rep_fx4.elapsed_seconds > 0 else float("inf")
    n, p_layer = spec.num_layers, spec.layer_bytes
    knee = min(1.0, max(0.0, 1.0 - tau_resident * b_host / (n * p_layer)))
    from .exponent_codec import CompressedModel

    ratio = CompressedModel.from_container(container, pin=False).ratio
    doc = {"model": args.model, "tokens": args.tokens, "top_k": args.top_k,
           "b_host": b_host, "b_dev": b_dev, "b_dec_pipeline": b_dec_pipeline, "b_fx4_fused": b_fx4_fused,
           "tau_comp_theory": tau_resident,
           "tau_comp_paged_run": tau_comp / 2, "tau_load_paged_run": tau_load / 2,
           "compression_ratio": ratio, "knee_alpha": knee,
           "note": "b_host/b_dev in raw-equivalent B/s (b_dev: the decoder alone; b_dec_pipeline: device-tier-only "
                   "paged stack, raw bytes over the step time beyond resident compute; b_fx4_fused: the FX4 device tier read in "
                   "place by the decode-into-GEMM kernel, raw bytes per second of step); tau per decode iteration "
                   "(N layers); knee per simulate.knee_alpha with the measured b_host and resident tau"}
    text = json.dumps(doc, indent=2)
    if getattr(args, "out", None):
        Path(args.out).write_text(text)
    print(text)
    return EXIT_OK


def _sim_config(args):
    """SimConfig from a `calibrate --out` file (measured on the GPU) or explicit flags."""
    from .simulate import calibrated_config

    measured = {}
    if args.calibration:
        measured = json.loads(Path(args.calibration).read_text())
    for key in ("b_dev", "b_host", "tau_comp_theory", "compression_ratio"):
        v = getattr(args, key, None)
        if v is not None:
            measured[key] = v
    missing = [k for k in ("b_dev", "b_host", "tau_comp_theory") if k not in measured]
    if missing:
        from .errors import ConfigError

        raise ConfigError(f"need {missing}: pass --calibration (from `calibrate --out`) or the flags")
    return calibrated_config(_spec(args), measured, batch_size=args.tokens, max_new_tokens=args.iterations,
                             kv_bytes_per_token=args.kv_bytes_per_token, context_start=args.context_start)


def cmd_simulate(args) -> int:
    """simulate.simulate_decode at a fixed alpha (cli.py:166-174)."""
    from .simulate import simulate_decode, write_samples_csv

    samples = simulate_decode(_sim_config(args), args.alpha)
    write_samples_csv(samples, args.csv)
    print(f"wrote {args.csv}: {len(samples)} iterations at alpha={args.alpha}")
    return EXIT_OK


def cmd_sweep_alpha(args) -> int:
    """simulate.sweep_alpha over a residency grid + the closed-form knee (cli.py:177-189)."""
    from .simulate import knee_alpha, sweep_alpha, write_sweep_csv

    sim = _sim_config(args)
    l = sim.spec.experts_per_layer
    grid = [m / l for m in range(1, l + 1)] if args.grid is None else [float(x) for x in args.grid.split(",")]
    rows = sweep_alpha(sim, grid)
    write_sweep_csv(rows, args.csv)
    print(f"wrote {args.csv}: {len(rows)} grid points, closed-form knee alpha*={knee_alpha(sim):.4f}")
    return EXIT_OK


def cmd_plan(args) -> int:
    """The planner's closed loop over the calibrated model (cli.py:192-208)."""
    from .residency import PlannerState
    from .simulate import check_trace_safety, run_control_loop, write_trace_csv

    sim = _sim_config(args)
    l = sim.spec.experts_per_layer
    state = PlannerState(experts_per_layer=l, device_experts=max(1, min(l, args.m0)), cooldown=args.cooldown,
                         io_balance=args.io_balance == "on")
    _, trace = run_control_loop(sim, state)
    check_trace_safety(sim, trace)
    write_trace_csv(trace, args.csv)
    adjustments = sum(1 for row in trace if row.adjusted)
    print(f"wrote {args.csv}: {len(trace)} iterations, {adjustments} adjustments, final alpha={trace[-1].alpha:.4f}")
    return EXIT_OK


def _sim_args(p):
    _model_args(p)
    p.add_argument("--calibration", help="JSON written by `calibrate --out` (b_host, b_dev, tau_comp_theory)")
    p.add_argument("--b-dev", dest="b_dev", type=float)
    p.add_argument("--b-host", dest="b_host", type=float)
    p.add_argument("--tau-comp", dest="tau_comp_theory", type=float)
    p.add_argument("--compression-ratio", dest="compression_ratio", type=float)
    p.add_argument("--tokens", type=int, default=256, help="batch size (tokens per decode step)")
    p.add_argument("--iterations", type=int, default=64)
    p.add_argument("--kv-bytes-per-token", type=int, default=0)
    p.add_argument("--context-start", type=int, default=0)
    p.add_argument("csv", help="output CSV")


def build_parser():
    p = argparse.ArgumentParser(prog="python -m paper_2604_02715_b200", description=__doc__.split("\n\n")[0])
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate", help="write a synthetic bf16 weight container (reference bytes)")
    g.add_argument("out")
    g.add_argument("--force", action="store_true")
    _model_args(g)
    g.set_defaults(fn=cmd_generate)
    c = sub.add_parser("compress", help="exponent-Huffman container (XPGC, reference bytes)")
    c.add_argument("infile")
    c.add_argument("out")
    c.add_argument("--force", action="store_true")
    c.set_defaults(fn=cmd_compress)
    v = sub.add_parser("verify", help="byte-compare a compressed container against the raw one")
    v.add_argument("infile")
    v.add_argument("compressed")
    v.set_defaults(fn=cmd_verify)
    r = sub.add_parser("run", help="GPU streamed run vs GPU resident baseline with ordering validation")
    _model_args(r)
    r.add_argument("--container", help="run on this XPGW file (mmap ingest) instead of a generated model")
    r.add_argument("--tokens", type=int, default=4)
    r.add_argument("--top-k", type=int, default=2)
    r.add_argument("--iterations", type=int, default=3)
    r.add_argument("--alpha", type=float, default=None, help="device-tier share (compressed in HBM)")
    r.add_argument("--mode", choices=["threaded", "sequential"], default="threaded")
    r.add_argument("--host-codec", action="store_true", help="page exponent-Huffman records over PCIe")
    r.add_argument("--seeds", type=int, default=1)
    r.add_argument("--out")
    r.set_defaults(fn=cmd_run)
    k = sub.add_parser("calibrate", help="measure the simulator's inputs on this GPU")
    _model_args(k)
    k.add_argument("--tokens", type=int, default=256)
    k.add_argument("--top-k", type=int, default=2)
    k.add_argument("--out", help="also write the measurements here (input of simulate/sweep-alpha/plan)")
    k.set_defaults(fn=cmd_calibrate)
    sm = sub.add_parser("simulate", help="the reference's decode model at a fixed alpha, calibrated inputs")
    _sim_args(sm)
    sm.add_argument("--alpha", type=float, default=0.25)
    sm.set_defaults(fn=cmd_simulate)
    sw = sub.add_parser("sweep-alpha", help="steady-state tau_load over a residency grid + knee alpha*")
    _sim_args(sw)
    sw.add_argument("--grid", help="comma-separated alphas (default m/L, m = 1..L)")
    sw.set_defaults(fn=cmd_sweep_alpha)
    pl = sub.add_parser("plan", help="the residency planner's closed loop over the calibrated model")
    _sim_args(pl)
    pl.add_argument("--m0", type=int, default=1, help="initial device-tier experts per layer")
    pl.add_argument("--cooldown", type=int, default=20)
    pl.add_argument("--io-balance", choices=["on", "off"], default="on")
    pl.set_defaults(fn=cmd_plan)
    return p


def main(argv=None) -> int:
    from .errors import ConfigError, OutOfRangeError, TruncatedStreamError, XpgError

    args = build_parser().parse_args(argv)
    try:
        return args.fn(args)
    except (ConfigError, OutOfRangeError) as exc:
        print(f"configuration error: {exc}", file=sys.stderr)
        return EXIT_VALIDATION
    except TruncatedStreamError as exc:
        print(f"corrupt container: {exc}", file=sys.stderr)
        return EXIT_IO
    except (OSError, XpgError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
