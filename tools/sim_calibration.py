"""Check the performance models against a measured budget sweep.

    python tools/sim_calibration.py --calibration gpurun_out/.../calib.json \
        --sweep profiles/r2_sweep_budget_mixtral.jsonl [--config mixtral] [--b-fused GBPS]

For every sweep point (device-tier and pinned experts per layer as the planner chose them)
it prints the reference model's prediction (simulate.predict_tiered: max(tau_comp, N x
tau_layer), simulate.py:96-146, fed with b_host, b_dev, tau_comp measured by ``calibrate``)
and this implementation's SM-sharing model (simulate.predict_sm_shared), each with its
relative error against the measured tok/s.  One JSON line per point, then a summary line.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SHAPES = {"mixtral": (8, 8, 4096, 14336), "qwen3": (8, 128, 2048, 768), "dsv3": (8, 32, 7168, 2048)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--calibration", required=True)
    ap.add_argument("--sweep", required=True)
    ap.add_argument("--config", default="mixtral")
    ap.add_argument("--b-fused", type=float, default=None, help="decode-into-GEMM raw-equivalent GB/s")
    ap.add_argument("--b-dec", type=float, default=None, help="in-pipeline decoder raw-equivalent GB/s")
    ap.add_argument("--host-exposed", type=float, default=None,
                    help="share of the link time an SM-bound step exposes (default budget.HOST_EXPOSED)")
    args = ap.parse_args()
    from paper_2604_02715_b200 import ModelSpec
    from paper_2604_02715_b200 import simulate as S
    from paper_2604_02715_b200.budget import HOST_EXPOSED

    cal = json.load(open(args.calibration))
    spec = ModelSpec(*SHAPES[args.config])
    worst = {"reference_model": 0.0, "sm_shared_model": 0.0}
    with open(args.sweep) as fh:
        points = [json.loads(l) for l in fh if l.strip()]
    for p in points:
        c = S.calibrated_config(spec, cal, batch_size=int(p.get("T", cal.get("tokens", 256))))
        dev, pin = float(p.get("device_tier_per_layer", 0)), float(p.get("pinned_per_layer", 0))
        ref = S.predict_tiered(c, dev, pin)
        b_dec = args.b_dec * 1e9 if args.b_dec else cal.get("b_dec_pipeline")
        fused = p.get("device_format") in ("fx4", "mixed") and p.get("fused_decode")
        b_fused = (args.b_fused * 1e9 if args.b_fused else cal.get("b_fx4_fused")) if fused else None
        fx = p.get("fx4_per_layer") if p.get("device_format") == "mixed" else None
        ours = S.predict_sm_shared(c, dev, pin, b_dec=b_dec, b_fused=b_fused, fx4_per_layer=fx,
                                   host_exposed=HOST_EXPOSED if args.host_exposed is None else args.host_exposed)
        meas = float(p["tok_s"])
        row = {"budget": p.get("budget"), "device_format": p.get("device_format", "huffman"), "fx4_per_layer": fx,
               "device_per_layer": dev, "pinned_per_layer": pin, "measured_tok_s": meas,
               "reference_model_tok_s": ref["tok_s"], "reference_model_err": ref["tok_s"] / meas - 1,
               "sm_shared_model_tok_s": ours["tok_s"], "sm_shared_model_err": ours["tok_s"] / meas - 1,
               "sm_shared_bound": ours["bound"]}
        worst["reference_model"] = max(worst["reference_model"], abs(row["reference_model_err"]))
        worst["sm_shared_model"] = max(worst["sm_shared_model"], abs(row["sm_shared_model_err"]))
        print(json.dumps(row))
    print(json.dumps({"summary": "max |relative error| over the sweep", **worst,
                      "inputs": {k: cal[k] for k in ("b_host", "b_dev", "b_dec_pipeline", "b_fx4_fused", "tau_comp_theory")
                                 if k in cal}}))


if __name__ == "__main__":
    main()
