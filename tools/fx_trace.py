"""Per-stage hand-off timeline of the FX4 decode-into-GEMM kernel (CTA 0, first unit, last
gate/up launch), from a trace build:

    python tools/fx_trace_build.py > /tmp/moe_gemm_dec.cu
    tools/micro/ab/build_variant.sh trace /tmp/moe_gemm_dec.cu
    XPGB_LIB_PATH=tools/micro/ab/trace/libxpgb.so python tools/fx_trace.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

SLOTS = ["B issue", "MMA B ready", "MMA A ready", "MMA commit", "C issue", "dec C ready", "dec C released",
         "dec A free", "dec A written"]


def main():
    import numpy as np
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200._lib import lib
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    spec = X.ModelSpec(2, 8, 4096, 14336)
    T = 256
    fwd = X.ForwardSpec(T, 2, 7)
    container = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(spec, backends, alpha=1.0), backends)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((T, 4096), dtype=np.float32)).cuda()
    runner = X.StreamedRunner(spec, hier, fwd, fused_decode=True, device_format="fx4")
    runner.run(2, acts=x.clone())
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 640)()
    lib().xpgb_debug_fx_trace.argtypes = [C.c_void_p]
    assert lib().xpgb_debug_fx_trace(C.cast(buf, C.c_void_p)) == 0
    t = np.array(buf, dtype=np.int64).reshape(10, 64)[:9]
    t0 = t[4, 0]
    rel = t - t0
    print("stage " + " ".join(f"{s[:12]:>13s}" for s in SLOTS))
    for kb in list(range(0, 8)) + list(range(56, 64)):
        print(f"{kb:5d} " + " ".join(f"{v:13d}" for v in rel[:, kb]))
    d = np.diff(t, axis=1)
    print("mean clocks per stage (steady, stages 8..63):", {SLOTS[i]: float(d[i, 8:].mean()) for i in range(9)})
    lag = {"C issue -> dec C ready": float((t[5] - t[4])[8:].mean()),
           "dec C ready -> released": float((t[6] - t[5])[8:].mean()),
           "released -> A free": float((t[7] - t[6])[8:].mean()),
           "A free -> A written": float((t[8] - t[7])[8:].mean()),
           "A written -> MMA A ready": float((t[2] - t[8])[8:].mean()),
           "MMA B ready -> A ready": float((t[2] - t[1])[8:].mean()),
           "MMA A ready -> commit": float((t[3] - t[2])[8:].mean()),
           "B issue -> MMA B ready": float((t[1] - t[0])[8:].mean())}
    print("mean lags (clocks):", lag)


if __name__ == "__main__":
    main()
