"""GPU exponent-decoder throughput on expert-shaped tensors (bf16 N(0, 0.02)).

    python tools/profile_codec.py [--values 117440512] [--chunk 1024]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--values", type=int, default=117_440_512)  # Mixtral gate/up tensor
    ap.add_argument("--chunk", type=int, default=256)
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2604_02715_b200 import exponent_codec as XC
    from paper_2604_02715_b200._lib import call, lib

    n = args.values
    w = torch.randn(n, device="cuda").mul_(0.02).to(torch.bfloat16).view(torch.int16).cpu().numpy().view("<u2")
    t = XC.build_table(XC.build_histogram(w))
    ct = XC.compress(w, t, chunk=args.chunk)
    rec = XC._record(ct, t)
    d_rec = torch.from_numpy(rec).cuda()
    out = torch.empty(n, dtype=torch.int16, device="cuda")
    lengths = t.lengths_array()
    s = torch.cuda.current_stream().cuda_stream

    def once():
        call("xpgb_codec_decode", C.c_void_p(d_rec.data_ptr()), C.c_uint64(n), C.c_uint64(len(ct.exponent_bitstream)),
             args.chunk, lengths.ctypes.data_as(C.POINTER(C.c_uint8)), C.c_void_p(out.data_ptr()), C.c_void_p(s))

    once()
    torch.cuda.synchronize()
    ok = out.cpu().numpy().view("<u2").tobytes() == w.tobytes()
    # hold the GPU busy ~0.5 s first: short launches on an idle GPU time its clock ramp
    warm = torch.empty(1 << 28, dtype=torch.float32, device="cuda")
    t_end = torch.cuda.Event(enable_timing=True)
    import time as _t
    t0 = _t.time()
    while _t.time() - t0 < 0.5:
        warm.mul_(1.0001)
        once()
    torch.cuda.synchronize()
    del warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.reps
    print(json.dumps({"decoder": "v1" if os.environ.get("XPGB_DECODER") == "1" else "v2", "values": n,
                      "chunk": args.chunk, "exact": ok, "ms": ms, "out_GBps": 2 * n / ms / 1e6,
                      "in_GBps": rec.size / ms / 1e6, "algo_GBps": (rec.size + 2 * n) / ms / 1e6,
                      "ratio": ct.compressed_bytes / (2 * n),
                      "bits_per_exponent": ct.exponent_bit_count / n}))


if __name__ == "__main__":
    main()
