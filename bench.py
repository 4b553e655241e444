#!/usr/bin/env python
"""Benchmark: MoE decode tokens/s at a fixed expert-HBM budget, page-in GB/s, exposed transfer %.

Workload (BASELINE.json configs[1]): Mixtral-8x7B-shaped MoE stack -- 8 layers, 8 experts,
top-2, hidden 4096, ffn 14336, bf16 weights from the reference generator (model.py:205-214),
one B200, 25% of the expert bytes in HBM.  The budget counts everything the path keeps in HBM
for expert weights: ring blocks, the compressed device tier, pinned experts, shared experts,
the codec's staging buffers and the device-resident chunk index (``expert_hbm_footprint``).
By default it is spent FluxMoE-style by the budget planner (budget.plan_residency): a
one-expert sub-layer ring, experts compressed in HBM (device tier), the rest streamed from
pinned host memory as exponent-Huffman records over PCIe and decoded on the GPU; ``--tiering
ring`` keeps the reference's 2-layer ring.  A step = one decode iteration of T=256 tokens
through all 8 layers.  Every timed run is checked for page faults and ordering violations;
the line is not printed when one is found.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

--gpus N without torchrun re-launches itself under torch.distributed.run with N ranks.
--impl reference times the reference algorithm's CPU path (the oracle port in
oracle/cpu_reference.py) on the host cores: each step is a bounded, really timed sample (one
layer's page-in plus the per-token forward of a few tokens of the step), and the line's
value extrapolates it linearly to the workload (8 layers x 256 tokens).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))

CONFIGS = {
    "mixtral": dict(N=8, L=8, H=4096, F=14336, k=2, T=256,
                    name="Mixtral-8x7B-shaped MoE stack (8 layers, 8 experts, top-2, hidden 4096, ffn 14336)"),
    "qwen3": dict(N=8, L=128, H=2048, F=768, k=8, T=256,
                  name="Qwen3-30B-A3B-shaped MoE stack (8 of 48 layers, 128 experts, top-8, hidden 2048, ffn 768)"),
    "tiny": dict(N=4, L=8, H=256, F=512, k=2, T=256,
                 name="tiny synthetic MoE (4 layers, 8 experts, top-2, hidden 256, ffn 512)"),
    # one GPU = rank 0 of 8-way expert parallelism: its 32-expert shard + the replicated shared
    # expert, routing the 8 x 256 global tokens (the all-to-all has no peer on one GPU)
    "dsv3": dict(N=8, L=256, H=7168, F=2048, k=8, T=256, S=1, ep_virtual=8,
                 name="DeepSeek-V3-shaped MoE layers (8 layers, 256 routed + 1 shared expert, top-8, hidden 7168, "
                      "ffn 2048), rank 0 of 8-way expert parallelism on one B200"),
}
METRIC = "MoE decode tokens/sec at fixed expert-HBM budget (25%); page-in GB/s; exposed xfer %"
METRIC_PREFILL = "MoE prefill tokens/sec at fixed expert-HBM budget (25%); page-in GB/s; exposed xfer %"
SEED = 7


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_tensor_peak():
    """Sustained dense bf16 TFLOP/s (the GEMMs run inside a long step), else the recipe's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p.get("bf16_tflops_sustained") or p["bf16_tflops"]), "measured (sustained)"
    except Exception:
        return 1590.0, "fallback"


def ncu_traffic(config: str, tokens: int):
    """DRAM bytes (read + write) of one gate/up launch from the committed ncu --set full
    capture of this workload (profiles/), or None when none was taken for it."""
    path = {("mixtral", 256): os.path.join(ROOT, "profiles", "r2_ncu_gemm_T256_final.jsonl")}.get((config, tokens))
    try:
        for line in open(path):
            rec = json.loads(line)
            if "<1," in rec.get("kernel", "") or "<true" in rec.get("kernel", ""):
                return rec.get("traffic_bytes")
    except Exception:
        return None
    return None


def ncu_decoder_capture():
    """DRAM traffic vs algorithmic bytes of one decoder launch (Mixtral gate/up tensor) from
    the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "r2_ncu_dec2_final.jsonl")
    try:
        rec = json.loads(open(path).readline())
        n = 117_440_512  # values of the captured tensor (tools/profile_codec.py default)
        algo = n + n * 2.591 / 8 + n / 256 * 4 + 2 * n
        return {"dram_bytes": rec["dram_read"] + rec["dram_write"], "algorithmic_bytes": algo,
                "source": "profiles/r2_ncu_dec2_final.jsonl (k_exp_decode2, one 117.4M-value tensor, chunk 256)"}
    except Exception:
        return None


def parity_summary():
    """Per-config float parity against the oracle (north star: rel err <= 1e-2, stated per
    config), from the committed -m gpu run of tests/test_gpu_fullshape_*.py (XPGB_PARITY_LOG):
    worst per-layer rel-L2 (teacher-forced, reference-generator weights, T = 1/16/256 and a
    CTA-pair size), the free-running short stack, and the paged stack at the bench tiering."""
    path = os.path.join(ROOT, "profiles", "r2_parity_fullshape.jsonl")
    try:
        rows = [json.loads(l) for l in open(path) if l.strip()]
    except OSError:
        return None
    out = {}
    for r in rows:
        c = out.setdefault(r["config"], {"per_layer_max": 0.0})
        if r["case"].startswith(("layer", "stack_teacher")):
            c["per_layer_max"] = max(c["per_layer_max"], r["rel_l2"])
        elif r["case"].startswith("stack_free"):
            c["free_stack"] = {"case": r["case"], "rel_l2": r["rel_l2"]}
        elif r["case"].startswith("paged"):
            c["paged_stack"] = {"case": r["case"], "rel_l2": r["rel_l2"]}
    return {"tolerance": 1e-2, "metric": "rel-L2 vs oracle layer_forward (xpg pipeline.py:192-208)",
            "per_config": out, "source": "profiles/r2_parity_fullshape.jsonl"}


PROFILE_EVERY = 7  # odd: gate/up and down decoder launches alternate


def decoder_roofline(stats, steps, step_s, hbm_peak, hbm_src):
    """Roofline of the exponent decoder (the dominant kernel of a paged decode step): its
    algorithmic bytes per launch over its mean launch time, both over the timed run."""
    n = stats.get("launches", 0)
    if not n:
        return None
    per_launch = stats["algo_bytes"] / n
    ns = stats["kernel_ns"] / n
    ach = per_launch / ns  # bytes/ns == GB/s
    return {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "peak_source": hbm_src, "kernel": "k_exp_decode2 (exponent-Huffman -> bf16 into the ring, paged run; 65% of kernel time, profiles/r2_launches_bench_mixtral.json)",
            "algorithmic_bytes_per_launch": per_launch, "avg_launch_us": ns / 1e3,
            "launches_per_step": n / steps, "kernel_time_per_step_ms": stats["kernel_ns"] / steps / 1e6,
            "step_ms": step_s * 1e3 / steps,
            "note": "launches overlap each other (two kinds, host and device tiers) and the GEMMs, so a launch's "
                    "time includes sharing the SMs; standalone the kernel reaches ~1,450-1,540 GB/s of bf16 output "
                    "on a 117M-value tensor, bound by the per-stream decode chain (profiles/r2_decoder_experiments.md)",
            "traffic": decoder_traffic(per_launch), "traffic_capture": ncu_decoder_capture()}


def decoder_traffic(algo_bytes):
    """DRAM bytes of a decoder launch with `algo_bytes` algorithmic bytes, scaled from the
    committed ncu --set full capture of one launch (DRAM / algorithmic = 0.89 there: the
    bitstream words a thread reads twice at chunk edges hit L2, and part of the output is still
    in L2 when the capture ends)."""
    cap = ncu_decoder_capture()
    if not cap:
        return None
    return algo_bytes * cap["dram_bytes"] / cap["algorithmic_bytes"]


def fused_roofline(stats, steps, hbm_peak, hbm_src):
    """Roofline of the decode-into-GEMM kernel: the compressed record bytes each launch reads in
    place (its DRAM traffic is those bytes + the activation rows, ncu: profiles/r2_ncu_fused_fx4_tmem.jsonl)
    over its mean launch time."""
    n = stats.get("launches", 0)
    if not n:
        return None
    per_launch = stats["record_bytes"] / n
    ns = stats["kernel_ns"] / n
    ach = per_launch / ns
    return {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "peak_source": hbm_src,
            "kernel": "k_moe_gemm_dec (decode-into-GEMM: device-tier records expanded into the UMMA tiles in smem)",
            "algorithmic_bytes_per_launch": per_launch, "avg_launch_us": ns / 1e3, "launches_per_step": n / steps,
            "kernel_time_per_step_ms": stats["kernel_ns"] / steps / 1e6,
            "note": "algorithmic bytes = the compressed records read in place (activation rows excluded)",
            "traffic": fused_traffic(per_launch)}


def fused_traffic(record_bytes):
    """DRAM bytes of a decode-into-GEMM launch that reads `record_bytes` of FX4 records, from the
    committed ncu --set full capture of a Mixtral gate/up launch (8 experts' records read in place:
    DRAM read + write over record bytes -- the activation re-reads and escape bytes on top)."""
    path = os.path.join(ROOT, "profiles", "r2_ncu_fused_fx4_tmem.jsonl")
    try:
        rec = json.loads(open(path).readline())
        n = 2 * 4096 * 14336
        captured = 8 * (n + n // 2 + 4 * (n // 256 + 1))  # 8 experts' FX4 gate/up records (no escapes)
        return record_bytes * (rec["dram_read"] + rec["dram_write"]) / captured
    except Exception:
        return None


def gemm_roofline(kind, bytes_, ns, rows, H, F, hbm_peak, hbm_src, tc_peak, tc_src):
    """Roofline of one grouped-GEMM launch: HBM-bound (weights dominate) at decode sizes,
    tensor-bound once the rows per expert make the contraction compute-heavy."""
    flops = 2.0 * rows * H * (2 * F if kind == "gate_up" else F)
    t = ns * 1e-9 if ns else 0.0
    if bytes_ and flops / bytes_ > tc_peak * 1e12 / (hbm_peak * 1e9):
        ach = flops / t / 1e12 if t else 0.0
        return {"bound": "tensor", "achieved": ach, "peak": tc_peak, "unit": "TFLOP/s",
                "frac": ach / tc_peak, "peak_source": tc_src, "flops_per_launch": flops,
                "algorithmic_bytes_per_launch": bytes_, "avg_launch_us": ns / 1e3}
    ach = bytes_ / t / 1e9 if t else 0.0
    return {"bound": "hbm", "achieved": ach, "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
            "peak_source": hbm_src, "algorithmic_bytes_per_launch": bytes_, "flops_per_launch": flops,
            "avg_launch_us": ns / 1e3}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms while active."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 7:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for name, val in zip(names, parts[3:7]):
                    if val.lower().startswith("active"):
                        reasons.add(name)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def h2d_peak_gbps(torch, device: int) -> float:
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    best = 0.0
    for i in range(6):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        d.copy_(h, non_blocking=True)
        e.record()
        e.synchronize()
        if i:
            best = max(best, n / (s.elapsed_time(e) * 1e-3) / 1e9)
    del h, d
    return best


def spawn_ranks(args) -> int:
    """bench.py --gpus N without torchrun: re-launch under torch.distributed.run with N ranks
    (one per GPU).  Fewer visible GPUs than N is an error unless --oversubscribe, which puts
    ranks round-robin on the GPUs there are (a test of the N-rank path, not a scaling number;
    the line says so)."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus and not args.oversubscribe:
        raise SystemExit(f"bench: --gpus {args.gpus} but only {have} GPU(s) visible "
                         "(--oversubscribe runs the ranks on shared GPUs)")
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_setup(oversubscribe: bool = False):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if oversubscribe:
            # ranks share GPUs: NCCL refuses two ranks on one device, so the plumbing (barrier,
            # max over ranks) runs on gloo; the EP data path uses peer windows (CUDA IPC)
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)  # one rank per GPU, bound before NCCL picks a device
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def max_over_ranks(torch, world: int, value: float, device: int) -> float:
    if world == 1:
        return value
    import torch.distributed as dist

    on_gpu = dist.get_backend() == "nccl"
    t = torch.tensor([value], dtype=torch.float64, device=f"cuda:{device}" if on_gpu else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def cpu_baseline(cfg, words, sample_tokens: int, container=None):
    from oracle import cpu_reference  # checker / baseline only

    if cfg.get("ep_virtual"):
        # the reference has no expert parallelism: one process pages the whole model; the
        # sample's experts are drawn from this rank's shard payload (same distribution)
        from paper_2604_02715_b200.geometry import ExpertTensorId, TensorKind

        cnt = container.spec.experts_per_layer
        tw = lambda layer, e, kind: container.tensor_words(ExpertTensorId(layer, (e - 1) % cnt + 1, TensorKind(kind)))
        sw = None
        if container.shared is not None:
            sw = lambda kind: container.shared.words[container.shared.offset(1, 1, kind) // 2:][
                :container.spec.value_count(kind)]
        r = cpu_reference.decode_rate_sampled(tw, cfg["N"], cfg["L"], cfg["H"], cfg["F"], cfg["T"], cfg["k"], SEED,
                                              sample_tokens, shared_words=sw)
        return {
            "value": r["tok_s"], "unit": "tokens/s", "cores": r["threads"], "kind": "port",
            "sample": (f"oracle/cpu_reference.py decode_rate_sampled: reference single-process path over the whole "
                       f"model (no expert parallelism in the reference): page-in of the {r['fetched_experts']} experts "
                       f"{sample_tokens} tokens route to, scaled to {cfg['L']} ({r['fetch_s']:.2f}s/layer), per-token "
                       f"forward incl. shared expert ({r['compute_s']:.2f}s), extrapolated to {cfg['N']} layers x "
                       f"T={cfg['T']}"),
        }
    r = cpu_reference.decode_rate(words, cfg["N"], cfg["L"], cfg["H"], cfg["F"], cfg["T"], cfg["k"], SEED,
                                  sample_tokens)
    return {
        "value": r["tok_s"], "unit": "tokens/s", "cores": r["threads"], "kind": "port",
        "sample": (f"oracle/cpu_reference.py: one layer page-in ({cfg['L']} experts, host copy {r['fetch_s']:.2f}s) "
                   f"+ reference per-token forward on {sample_tokens} tokens ({r['compute_s']:.2f}s), "
                   f"extrapolated to {cfg['N']} layers x T={cfg['T']}"),
    }


def run_reference_arm(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np

    from oracle import cpu_reference, xpg_oracle as O

    threads = os.cpu_count() or 1
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    sample = args.ref_sample_tokens
    H, F = cfg["H"], cfg["F"]
    layer_words = cfg["L"] * (O.sigma(H, F, 1) + O.sigma(H, F, 2)) // 2
    rng = np.random.default_rng(SEED)
    if layer_words * 2 <= (4 << 30):
        # weights of layer 1 (all the sample touches): the reference generator's first draws
        # (numpy's PCG64 stream decoded in parallel segments; data setup, outside the timing)
        from paper_2604_02715_b200.geometry import _fill_normal_bf16

        words = np.empty(layer_words, dtype=np.uint16)
        _fill_normal_bf16(SEED, [words])
        step_fn = lambda: cpu_reference.decode_rate(words, cfg["N"], cfg["L"], H, F, cfg["T"], cfg["k"], SEED, sample)
    else:
        # a layer too large to hold (DSv3: 22.5 GB): draw only the experts the sample routes to
        # (same distribution), time their page-in and scale it to the layer (decode_rate_sampled)
        routed = sorted({int(j) for j in O.route(SEED, sample, 1, cfg["L"], cfg["k"]).reshape(-1)})
        n1, n2 = O.sigma(H, F, 1) // 2, O.sigma(H, F, 2) // 2
        pool = {j: (O.f32_to_bf16(rng.standard_normal(n1, dtype=np.float32) * O.WEIGHT_STD),
                    O.f32_to_bf16(rng.standard_normal(n2, dtype=np.float32) * O.WEIGHT_STD)) for j in routed}
        shared = None
        if cfg.get("S"):
            sh = (O.f32_to_bf16(rng.standard_normal(n1, dtype=np.float32) * O.WEIGHT_STD),
                  O.f32_to_bf16(rng.standard_normal(n2, dtype=np.float32) * O.WEIGHT_STD))
            shared = lambda kind: sh[kind - 1]
        step_fn = lambda: cpu_reference.decode_rate_sampled(lambda layer, j, kind: pool[j][kind - 1], cfg["N"],
                                                            cfg["L"], H, F, cfg["T"], cfg["k"], SEED, sample,
                                                            shared_words=shared)
    samples = []
    for i in range(args.warmup + args.steps):
        w0 = time.perf_counter()
        r = step_fn()
        wall = time.perf_counter() - w0
        if i >= args.warmup:
            samples.append((wall, r))
    # each step is a real, timed bounded sample: one layer's page-in (all L experts copied into
    # the arena, storage.py:235-243) + the reference per-token forward of `sample` tokens of
    # the step (pipeline.py:192-208).  The workload's rate is the linear extrapolation of the
    # measured costs: every layer does the same work, and a step is N x (fetch + T x per-token).
    fetch = sum(r["fetch_s"] for _, r in samples) / len(samples)
    per_tok = sum(r["per_token_s"] for _, r in samples) / len(samples)
    full_step = cfg["N"] * (fetch + cfg["T"] * per_tok)
    value = cfg["T"] / full_step
    wall_ms = 1e3 * sum(w for w, _ in samples) / len(samples)
    sample_desc = (f"per step: layer-1 page-in of {cfg['L']} experts ({fetch:.2f}s) + reference per-token forward "
                   f"of {sample} of the step's {cfg['T']} tokens ({per_tok:.2f}s/token), really timed; value = "
                   f"T / (N x (fetch + T x per-token)) for N={cfg['N']} layers, T={cfg['T']} "
                   f"(oracle/cpu_reference.py, a port of xpg pipeline.py/storage.py)")
    line = {
        "impl": "reference", "metric": METRIC_PREFILL if args.prefill else METRIC, "value": value,
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": wall_ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generator, seed 7)",
        "config": {"workload": cfg["name"], "tokens_per_step": cfg["T"], "top_k": cfg["k"], "layers": cfg["N"]},
        "sample": {"tokens": sample, "layers": 1, "measured_ms_per_sample": wall_ms,
                   "fetch_s_per_layer": fetch, "per_token_s_per_layer": per_tok,
                   "extrapolated_ms_per_full_step": 1e3 * full_step,
                   "measured_tok_s_at_sample_batch": sample / (cfg["N"] * (fetch + sample * per_tok))},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": sample_desc},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


_T0 = time.time()
_VERIFIED = []


def verify(what: str, fault, violations) -> None:
    """A timed run must have done all its work: a device page fault makes every kernel of the
    step return early (only the copies would be timed), an ordering violation means a RAW/WAR
    hazard.  Either one aborts the bench before a number is printed."""
    if fault is not None or violations:
        raise SystemExit(f"bench: {what} is invalid: page_fault={fault!r} violations={list(violations)[:3]}")
    _VERIFIED.append(what)


def log(msg):
    mem = ""
    try:
        import torch

        if torch.cuda.is_available() and torch.cuda.is_initialized():
            free, total = torch.cuda.mem_get_info()
            mem = f" [HBM free {free / 2**30:.1f}/{total / 2**30:.1f} GiB]"
    except Exception:
        pass
    print(f"[bench {time.time() - _T0:7.1f}s] {msg}{mem}", file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="mixtral", choices=sorted(CONFIGS))
    ap.add_argument("--tokens", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None,
                    help="override the config's layer count (Qwen3-30B-A3B has 48; the default stack is 8)")
    ap.add_argument("--device-format", default="auto", choices=["auto", "huffman", "fx4", "mixed"],
                    help="device-tier records: exponent-Huffman decoded into the ring, FX4 read in place by "
                         "the decode-into-GEMM kernel, or mixed (every expert on the device tier, as many FX4 as "
                         "fit; auto: the planner's step model picks)")
    ap.add_argument("--budget", type=float, default=0.25,
                    help="expert-HBM budget as a fraction of the expert bytes (ring + codec buffers + shared)")
    ap.add_argument("--tiering", default="device", choices=["device", "ring"],
                    help="spend the budget on a compressed device tier + small ring (FluxMoE), or ring only")
    ap.add_argument("--prefill", action="store_true",
                    help="prefill regime: one step = a T-token prompt chunk through every layer (default T=8192)")
    ap.add_argument("--cpu-sample-tokens", type=int, default=16)  # ~10 s of host work at Mixtral shape
    ap.add_argument("--ref-sample-tokens", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-resident", action="store_true")
    ap.add_argument("--act-planes", type=int, default=2, choices=[1, 2],
                    help="activation planes of the decode-sized GEMMs: 2 = bf16 hi + lo (fp32-like, default), "
                         "1 = bf16 activations (half the MMAs; rel-L2 ~3e-3, inside the 1e-2 tolerance)")
    ap.add_argument("--no-timed-profile", action="store_true",
                    help="A/B only: time the paged run without its per-launch events (no kernel rooflines)")
    ap.add_argument("--ep", action="store_true", help="use the expert-parallel runner even at N=1")
    ap.add_argument("--transport", default="auto", choices=["auto", "p2p", "nccl"],
                    help="EP dispatch/combine: peer-memory scatter kernels (p2p), NCCL all_to_all, or p2p when "
                         "every peer window opens (auto)")
    ap.add_argument("--weights", default=None, choices=["reference", "fast"],
                    help="reference: the reference generator's bf16 weights (bit-identical, default when the "
                         "model's stream is <= 32 GB); fast: the same distribution drawn on the GPU (torch Philox)")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="--gpus N with fewer GPUs: run the N ranks on shared GPUs (tests the N-rank path)")
    ap.add_argument("--raw", action="store_true",
                    help="page raw bf16 over PCIe (the reference host tier) instead of exponent-Huffman records")
    args = ap.parse_args()
    args.host_codec = not args.raw
    if args.weights is None:
        c0 = CONFIGS[args.config]
        stream = c0["N"] * (c0["L"] + c0.get("S", 0)) * 6 * c0["H"] * c0["F"]  # bytes of the generator stream
        args.weights = "reference" if stream <= (32 << 30) and not c0.get("ep_virtual") else "fast"
    cfg = dict(CONFIGS[args.config])
    if args.prefill and not args.tokens:
        args.tokens = 8192
    if args.tokens:
        cfg["T"] = args.tokens
    if args.layers:
        cfg["N"] = args.layers
        name = cfg["name"]
        cfg["name"] = (name.replace("8 of 48 layers", f"{args.layers} of 48 layers") if "8 of 48 layers" in name
                       else name.replace("8 layers", f"{args.layers} layers"))
    if args.prefill and args.device_format == "auto":
        # prefill-sized groups run on the CTA-pair GEMMs, which read ring blocks: a device tier
        # is decoded into the ring there, where exponent-Huffman (smaller) is the better format
        args.device_format = "huffman"
    if args.impl == "reference":
        run_reference_arm(args, cfg)
        return

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world, rank, local = dist_setup(args.oversubscribe)
    if world != args.gpus and args.gpus > 1:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}")
    import numpy as np
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.device import kernel_launches

    torch.cuda.set_device(local)
    dev = local
    N, L, H, F, k, T = cfg["N"], cfg["L"], cfg["H"], cfg["F"], cfg["k"], cfg["T"]
    S = cfg.get("S", 0)
    spec = X.ModelSpec(N, L, H, F)
    G_virt = cfg.get("ep_virtual", 1) if world == 1 and not args.ep else 1
    T_run = G_virt * T  # rows the step routes (an EP rank routes the global batch)
    fwd = X.ForwardSpec(T_run, k, SEED)
    run_kw = {}
    cspec = spec
    if G_virt > 1:
        from paper_2604_02715_b200.expert_parallel import shard_bounds

        first, count = shard_bounds(L, G_virt)[0]
        cspec = X.ModelSpec(N, count, H, F)  # this rank's shard payload
        run_kw = {"expert_shard": (first, count), "shared_tokens": (0, T)}
    t0 = time.time()
    use_ep = world > 1 or args.ep
    if use_ep:
        from paper_2604_02715_b200.expert_parallel import ExpertParallelRunner, shard_bounds

        first, count = shard_bounds(L, world)[rank]
        # each rank holds only its expert shard (shard-local container order) in pinned memory
        shard = X.generate_fast_model(X.ModelSpec(N, count, H, F), SEED + 1000 * rank, device=dev,
                                      shared_experts=S)
        container = None
    elif args.weights == "reference":
        # the reference generator (model.py:205-214), bit-identical, decoded in parallel segments
        container = X.generate_synthetic_model(cspec, SEED + rank, shared_experts=S)
    else:
        container = X.generate_fast_model(cspec, SEED + rank, device=dev, shared_experts=S)
    gen_s = time.time() - t0
    log(f"model generated in {gen_s:.1f}s")
    if use_ep:
        group = None
        runner = ExpertParallelRunner(spec, None, fwd, rank, world, device=dev, group=group, shard_pool=shard.pinned,
                                      transport=args.transport,
                                      shared=shard.shared, host_codec=args.host_codec)
        ep_transport = ("scatter kernels into peer windows over NVLink (CUDA IPC), epoch flags)"
                        if runner.transport == "p2p" else "NCCL all_to_all)") + (
                           f"; {runner.transport_note}" if runner.transport_note else "")
        shard_bytes = shard.spec.total_bytes + (shard.shared.total_bytes if shard.shared is not None else 0)
        m_dev = pinned_per_layer = 0
        if args.tiering == "device" and args.host_codec:
            # the same budget planner on this rank's shard (budget.plan_residency)
            from paper_2604_02715_b200.budget import plan_residency

            ceb = runner.device_tier_bytes(count) / (N * count) * 1.002
            sh_b = shard.shared.total_bytes if shard.shared is not None else 0
            plan = plan_residency(N, count, shard.spec.expert_bytes, ceb, args.budget * shard_bytes * 0.998,
                                  shared_bytes=sh_b, overhead_bytes=runner.ctx.hbm_bytes()["staging"])
            if plan.device_experts or plan.pinned_experts:
                runner.apply_plan(plan)
                m_dev, pinned_per_layer = plan.device_experts / N, plan.pinned_experts / N
        hbm = runner.ctx.hbm_bytes()
        budget = (hbm["ring"] + hbm["device_tier"]) / shard_bytes
        footprint = (hbm["ring"] + hbm["staging"] + hbm["device_tier"]) / shard_bytes
        ring_depth = runner.ctx._depth
    else:
        backends = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 55e9, 1 << 50)]
        hier = X.StorageHierarchy(container, None, X.plan_placement(cspec, backends), backends)
        raw_path = None
        if args.host_codec:
            # the reference host tier (raw bf16 over PCIe) on the same weights, for comparison
            raw_runner = X.StreamedRunner(spec, hier, fwd, mode="threaded", device=dev, **run_kw)
            xr = torch.from_numpy(X.initial_activations(spec, fwd, SEED + rank)).to(f"cuda:{dev}")
            raw_runner.run(max(1, args.warmup - 1), acts=xr)
            torch.cuda.synchronize()
            q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            q0.record()
            rrep_raw = raw_runner.run(args.steps, acts=xr)
            q1.record()
            torch.cuda.synchronize()
            raw_s = q0.elapsed_time(q1) * 1e-3
            raw_path = {"tok_s": T * args.steps / raw_s, "ms_per_step": 1e3 * raw_s / args.steps,
                        "page_in_gbps": rrep_raw.h2d_bytes / rrep_raw.elapsed_seconds / 1e9,
                        "exposed_xfer_pct": 100.0 * rrep_raw.stall_seconds / rrep_raw.elapsed_seconds}
            del raw_runner
            log(f"raw host tier: {raw_path['tok_s']:.1f} tok/s")
        if args.host_codec:
            from paper_2604_02715_b200.exponent_codec import CompressedModel

            t1 = time.time()
            hier.compressed = CompressedModel.from_container(container)
            log(f"packed compressed host pool: ratio {hier.compressed.ratio:.4f} "
                f"({hier.compressed.wire_bytes / 1e9:.2f} GB) in {time.time() - t1:.1f}s")
        runner = X.StreamedRunner(spec, hier, fwd, mode="threaded", device=dev, host_codec=args.host_codec, **run_kw)
        runner.ctx.set_activation_planes(args.act_planes)
        hbm = runner.ctx.hbm_bytes()
        expert_bytes = cspec.total_bytes + (container.shared.total_bytes if container.shared is not None else 0)
        # fixed expert-HBM budget (north star): HBM holding expert weights -- ring slots, the
        # compressed device tier, resident shared experts -- within args.budget of the expert
        # bytes (the reference's own accounting: window + alpha x compressed pool,
        # simulate.py:50-66).  --tiering device (default with the codec) spends the budget like
        # FluxMoE: a small sub-layer ring, and every byte left holds experts 1..m of each layer
        # compressed in HBM (decoded on-GPU into the ring), so only L-m experts per layer cross
        # PCIe; --tiering ring keeps the reference's ring-only geometry.  The codec's staging
        # buffers and device-resident chunk index are part of the footprint the budget bounds.
        eb = cspec.expert_bytes
        shared_b = container.shared.total_bytes if container.shared is not None else 0
        ring_blocks = (hbm["ring"] - shared_b) // eb
        # the codec's staging buffers and device-resident chunk index count inside the budget
        overhead = hbm["staging"]
        cap = args.budget * expert_bytes * 0.998 - shared_b - overhead  # margin: record sizes vary per expert
        m_dev = 0
        pinned_per_layer = 0
        dev_format, dev_fused, fx4_per_layer = "huffman", False, 0.0
        if args.tiering == "device" and args.host_codec:
            from paper_2604_02715_b200.budget import fx4_expert_bytes, plan_tiers

            Lc, Nl = cspec.experts_per_layer, cspec.num_layers
            ceb = runner.device_tier_bytes(Lc) / (Nl * Lc) * 1.002  # compressed expert (+ margin)
            plan = plan_tiers(Nl, Lc, eb, ceb, cap + shared_b + overhead, shared_bytes=shared_b,
                              overhead_bytes=overhead, device_format=args.device_format,
                              fx4_ceb=fx4_expert_bytes(cspec.hidden_dim, cspec.intermediate_dim) * 1.002,
                              units_per_expert=cspec.intermediate_dim // 128)
            if plan.device_experts or plan.pinned_experts:
                runner.apply_plan(plan)
                ring_blocks = min(plan.ring, ring_blocks) if plan.ring else ring_blocks
                m_dev = plan.device_experts / Nl
                pinned_per_layer = plan.pinned_experts / Nl
                dev_format, dev_fused = plan.device_format, plan.fused
                fx4_per_layer = plan.fx4_experts / Nl
        if not (m_dev or pinned_per_layer):
            ring_fit = int((cap + 1) // eb) & ~1
            if 2 <= ring_fit < ring_blocks:
                runner.ctx.set_ring_experts(ring_fit)
                ring_blocks = ring_fit
        hbm = runner.ctx.hbm_bytes()
        budget = (hbm["ring"] + hbm["device_tier"]) / expert_bytes
        footprint = (hbm["ring"] + hbm["staging"] + hbm["device_tier"]) / expert_bytes
        ring_depth = runner.ctx._depth
    x_host = X.initial_activations(spec, fwd, SEED + rank)
    x_dev = torch.from_numpy(x_host).to(f"cuda:{dev}")

    # ---- warm-up (untimed)
    log("warm-up")
    runner.run(args.warmup, acts=x_dev)
    torch.cuda.synchronize()
    barrier(world)

    # ---- timed: K decode steps, inputs resident in HBM, one pipelined session
    with ClockSampler(dev) as clocks:
        launches0 = kernel_launches()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        # light profile: events around 1 in 7 decoder / decode-into-GEMM launches (the kernel
        # rooflines below); per-launch events on every launch cost 1-18% of the step
        rep = runner.run(args.steps, acts=x_dev, profile=0 if args.no_timed_profile else PROFILE_EVERY)
        ev1.record()
        torch.cuda.synchronize()
        launches = kernel_launches() - launches0
    verify("timed paged run", rep.page_fault, rep.violations)
    barrier(world)
    elapsed = max_over_ranks(torch, world, ev0.elapsed_time(ev1) * 1e-3, dev)
    tokens_total = T * args.steps * world
    value = tokens_total / elapsed
    page_in_gbps = rep.h2d_bytes / rep.elapsed_seconds / 1e9
    exposed = rep.stall_seconds / rep.elapsed_seconds
    dec_stats = runner.ctx.decode_stats()  # every decoder launch of the timed run, events on its own stream
    fz_stats = runner.ctx.fused_stats()    # every decode-into-GEMM launch of the timed run

    log(f"timed paged run: {elapsed:.3f}s")
    # ---- e2e: the same metric through the public API with host buffers every step: a
    # serving session (StreamedRunner.open_session) fed from pinned host memory, each step's
    # output read back into pinned host memory; the next step's first layers prefetch while
    # the host holds the previous result (the EP runner has the same session API)
    e2e_steps = args.steps
    x_pin = torch.from_numpy(x_host).pin_memory()
    out_pin = torch.empty_like(x_pin).pin_memory()
    sess = runner.open_session(max_iterations=e2e_steps + 1, log=False)
    sess.step(x_pin, out=out_pin)  # session warm-up step (untimed)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_steps):
        out = sess.step(x_pin, out=out_pin)  # pinned H2D in, D2H out, every step
    e1.record()
    torch.cuda.synchronize()
    srep = sess.close()
    verify("e2e session", srep.page_fault, srep.violations)
    del sess  # the session holds the runner (and its HBM ring) alive
    e2e_elapsed = max_over_ranks(torch, world, e0.elapsed_time(e1) * 1e-3, dev)
    if use_ep:
        runner.close()  # peer windows: every rank unmaps, barrier, then frees its own
    e2e_value = T * e2e_steps * world / e2e_elapsed
    assert tuple(out.shape) == x_host.shape  # (deep synthetic stacks overflow by design)

    log(f"e2e: {e2e_elapsed:.3f}s")
    # ---- fully-resident comparator: same kernels, every page resident in HBM
    resident = {}
    kern = rep.kernels
    if not args.no_resident and not use_ep:
        del runner
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        model = X.ResidentModel(spec, container, device=dev, max_tokens=T_run, **run_kw)
        model.ctx.set_activation_planes(args.act_planes)
        model.run(args.warmup, fwd, x_dev)
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        _, rrep = model.run(args.steps, fwd, x_dev, profile=True)
        r1.record()
        torch.cuda.synchronize()
        verify("resident run", model.ctx.fault() if rrep.page_fault else None, [])
        rt = r0.elapsed_time(r1) * 1e-3
        resident = {"tok_s": T * args.steps / rt, "ms_per_step": 1e3 * rt / args.steps}
        kern = {n: getattr(rrep, n) for n in ("kern_gate_up_ns", "kern_down_ns", "kern_aux_ns", "gate_up_bytes",
                                                 "down_bytes", "down_splits", "active_experts")}
        kern = {"gate_up_ns": kern["kern_gate_up_ns"], "down_ns": kern["kern_down_ns"], "aux_ns": kern["kern_aux_ns"],
                "gate_up_bytes": kern["gate_up_bytes"], "down_bytes": kern["down_bytes"],
                "down_splits": kern["down_splits"], "active_experts": kern["active_experts"]}
        paged_kern = rep.kernels
        del model

    log("resident done")
    hbm_peak, peak_src = load_peaks()
    h2d_peak = h2d_peak_gbps(torch, dev)
    tc_peak, tc_src = load_tensor_peak()
    # local rows per launch, from the algorithmic bytes (a experts x sigma1 + rows x (H + F) x 2 B)
    a_per_layer = kern.get("active_experts", 0) / N
    rows = max(0.0, (kern.get("gate_up_bytes", 0) - a_per_layer * 4 * H * F) / (2 * (H + F)))
    roof = gemm_roofline("gate_up", kern.get("gate_up_bytes", 0), kern.get("gate_up_ns", 0), rows, H, F,
                         hbm_peak, peak_src, tc_peak, tc_src)
    roof_dn = gemm_roofline("down", kern.get("down_bytes", 0), kern.get("down_ns", 0), rows, H, F,
                            hbm_peak, peak_src, tc_peak, tc_src)
    roof.update({"kernel": "k_moe_gemm<gate_up> (tcgen05 grouped SwiGLU GEMM, resident run)",
                 "traffic": ncu_traffic(args.config, T_run), "rows_per_launch": rows,
                 "down": {k: roof_dn[k] for k in ("bound", "achieved", "peak", "unit", "frac", "avg_launch_us")}})
    roof["down"]["splits"] = kern.get("down_splits")
    # the dominant kernel of the paged step is the decoder when the codec tiers are on (ncu
    # launch list: profiles/r2_launches_bench_mixtral.json); the GEMM roofline rides along
    dec_roof = decoder_roofline(dec_stats, args.steps, elapsed, hbm_peak, peak_src)
    fz_roof = fused_roofline(fz_stats, args.steps, hbm_peak, peak_src)
    # the dominant kernel of the paged step: the decoder or the decode-into-GEMM kernel,
    # whichever took more device time in the timed run
    if fz_roof is not None and (dec_roof is None or fz_stats["kernel_ns"] > dec_stats.get("kernel_ns", 0)):
        if dec_roof is not None:
            fz_roof["decoder"] = {k: dec_roof[k] for k in ("achieved", "frac", "avg_launch_us", "launches_per_step",
                                                          "kernel_time_per_step_ms")}
        dec_roof = fz_roof
    elif dec_roof is not None and fz_roof is not None:
        dec_roof["decode_into_gemm"] = {k: fz_roof[k] for k in ("achieved", "frac", "avg_launch_us",
                                                               "launches_per_step", "kernel_time_per_step_ms")}
    if dec_roof is not None:
        if roof.get("achieved"):  # EP runs have no resident comparator to time the GEMMs on
            dec_roof["gemm"] = roof
        roof = dec_roof

    line = {
        "metric": METRIC_PREFILL if args.prefill else METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": ("synthetic: bf16 weights from the reference generator (default_rng(7) N(0,0.02), bit-identical "
                 "to xpg model.py:205-214), N(0,1) activations" if args.weights == "reference" and not use_ep else
                 "synthetic: random-init N(0,0.02) bf16 weights drawn on-GPU (torch Philox; the reference generator's "
                 "stream for this model is too long to draw per run), N(0,1) activations"),
        "config": {"workload": cfg["name"], "tokens_per_step": T, "top_k": k, "layers": N,
                   "expert_hbm_budget": args.budget,
                   "expert_hbm_footprint": round(footprint, 4),
                   "expert_hbm_weights": round(budget, 4),
                   "footprint_counts": "ring + pinned + shared + compressed device tier + staging buffers + "
                                       "device-resident chunk index, / expert bytes",
                   "ring_blocks_per_kind": int(ring_blocks) if not use_ep else None,
                   "device_tier_experts_per_layer": round(m_dev, 3),
                   "pinned_experts_per_layer": round(pinned_per_layer, 3),
                   "device_tier_format": dev_format if not use_ep else "huffman",
                   "decode_into_gemm": bool(dev_fused) if not use_ep else False,
                   "fx4_experts_per_layer": round(fx4_per_layer, 3) if not use_ep else 0.0,
                   "activation_planes": args.act_planes,
                   "placement": ("2-layer ring" if use_ep or ring_blocks >= 2 * cspec.experts_per_layer else
                                 f"sub-layer ring of {ring_blocks} expert blocks per kind ({ring_depth} window(s) "
                                 f"in flight of {max(1, ring_blocks // ring_depth)} expert(s))") + (
                       f", {m_dev:.2f} experts per layer compressed in HBM (device tier, alpha="
                       f"{m_dev / (count if use_ep else cspec.experts_per_layer):.3f}, spread over the ring windows), "
                       f"the rest host" if m_dev else
                       ", host-only (alpha=0)") + (
                       ", exponent-Huffman records over PCIe decoded on-GPU into the ring (lossless)"
                       if args.host_codec else "") + (
                       (f"; device tier mixed: {fx4_per_layer:.2f} experts per layer in FX4 records read in place "
                        f"by the decode-into-GEMM kernel, the rest exponent-Huffman decoded into the ring"
                        if dev_format == "mixed" else
                        "; device tier in FX4 records read in place by the decode-into-GEMM kernel")
                       if (not use_ep and dev_fused) else ""),
                   "l2": ("inputs larger than L2 (126 MB): each step reads %.1f GB of expert weights -- %.2f GB of "
                          "records over PCIe, %.2f GB of bf16 decoded on-GPU from HBM records, the rest pinned/ring"
                          % (cspec.total_bytes / 1e9, rep.h2d_bytes / args.steps / 1e9,
                             rep.decoded_bytes / args.steps / 1e9))},
        "verified": {"runs": list(_VERIFIED), "page_fault": None, "ordering_violations": 0,
                     "note": "timed, e2e and resident runs checked for device page faults and RAW/WAR "
                             "ordering violations (bench aborts otherwise)"},
        "page_in": {"achieved_gbps": page_in_gbps, "peak_gbps": h2d_peak, "frac": page_in_gbps / h2d_peak if h2d_peak else None,
                    "bytes_per_step": rep.h2d_bytes / args.steps, "peak_how": "pinned 1 GiB cudaMemcpyAsync H2D, best of 5, this box",
                    "host_codec": bool(args.host_codec),
                    "raw_bytes_per_step": cspec.total_bytes if not use_ep else None,
                    "decoded_bytes_per_step": rep.decoded_bytes / args.steps,
                    "effective_raw_gbps": (cspec.total_bytes * args.steps / rep.elapsed_seconds / 1e9) if not use_ep else None},
        "exposed_xfer_pct": 100.0 * exposed,
        "war_wait_ms": rep.war_wait_seconds * 1e3,
        "roofline": roof,
        "resident": resident,
        "paged_over_resident": (value / world) / resident["tok_s"] if resident else None,
        "e2e": {"value": e2e_value, "unit": "tokens/s", "h2d_bytes_per_step": int(x_host.nbytes),
                "d2h_bytes_per_step": int(x_host.nbytes),
                "api": "StreamedRunner.open_session(...).step(pinned host acts)" if not use_ep else
                       "ExpertParallelRunner.open_session(...).step(pinned host acts)"},
        "parity": parity_summary(),
        "gpu_launches": launches,
        "clocks": clocks.summary(),
        "model_gen_s": gen_s,
    }
    if not args.no_resident and not use_ep and any(paged_kern.get(k) for k in ("gate_up_ns", "down_ns")):
        line["paged_kernels"] = paged_kern  # per-step events: only when the timed run profiles every launch
    if not use_ep and raw_path is not None:
        line["raw_host_tier"] = raw_path
    if use_ep:
        line["config"]["parallelism"] = f"ep{world} (experts sharded; dispatch/combine: {ep_transport}"
        if args.oversubscribe:
            import torch as _t

            line["config"]["oversubscribed"] = (f"{world} ranks on {_t.cuda.device_count()} GPU(s): tests the "
                                                f"{world}-rank path; not a scaling measurement")
        line["config"]["tokens_per_rank"] = T
    if G_virt > 1:
        line["config"]["parallelism"] = (f"rank 0 of ep{G_virt}: experts {run_kw['expert_shard'][0] + 1}.."
                                         f"{sum(run_kw['expert_shard'])} of {L} paged on this GPU, shared expert "
                                         f"replicated; routes the {T_run}-token global batch, applies the shared "
                                         f"expert to its own {T} tokens; all-to-all not timed (no peer on one GPU)")
        line["config"]["global_tokens_routed"] = T_run
    if S:
        line["config"]["shared_experts"] = S
    if rank == 0 and world == 1 and not args.no_cpu_baseline and container is not None:
        os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
        import numpy as np  # noqa: F811

        words = container.words[: cspec.layer_bytes // 2]
        line["cpu_baseline"] = cpu_baseline(cfg, words, args.cpu_sample_tokens, container)
    log("cpu baseline done")
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
