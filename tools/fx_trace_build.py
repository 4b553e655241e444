"""Make a trace build of the decode-into-GEMM kernel: clock64 stamps at every hand-off of CTA 0's
first unit (FX4, A tiles in TMEM, gate/up launches), read back by tools/fx_trace.py.

    python tools/fx_trace_build.py > /tmp/moe_gemm_dec.cu
    tools/micro/ab/build_variant.sh trace /tmp/moe_gemm_dec.cu
    XPGB_LIB_PATH=tools/micro/ab/trace/libxpgb.so python tools/fx_trace.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    src = open(os.path.join(ROOT, "paper_2604_02715_b200", "csrc", "moe_gemm_dec.cu")).read()

    def ins(after, code):
        nonlocal src
        assert src.count(after) == 1, after[:70]
        src = src.replace(after, after + code)

    src = src.replace("namespace xpgb {\n", "namespace xpgb {\n__device__ unsigned long long g_fx_trace[10][64];\n"
                      "#define FXTR(slot, cond) if (GU && FMT == 2 && blockIdx.x == 0 && u == (int)blockIdx.x && "
                      "(kb - kb0) < 64 && (cond)) g_fx_trace[slot][kb - kb0] = clock64();\n", 1)
    ins("          mbar_wait_backoff(&empty[stage], phase ^ 1);\n          uint8_t* sb = smem + stage * C::STAGE + C::B_OFF;",
        "\n          FXTR(0, true)")
    ins("        mbar_wait_role(&full[stage], phase, FMT >= 1 && (chunk & kFxSpinFlag));", "\n        FXTR(1, lane == 0)")
    ins("        if constexpr (FMT == 2) mbar_wait_role(&afull[ast], aph, chunk & kFxSpinFlag);", "\n        FXTR(2, lane == 0)")
    ins("          if constexpr (FMT == 2) umma_commit(&aempty[ast]);", "\n          FXTR(3, true)")
    ins("          mbar_wait_backoff(&cempty[cs], cph ^ 1);", "\n          FXTR(4, true)")
    ins("        mbar_wait(&cfull[fcs], fcph);", "\n        FXTR(5, threadIdx.x == 192)")
    ins("        if (lane == 0) mbar_arrive(&cempty[fcs]);", "\n        FXTR(6, threadIdx.x == 192)")
    ins("        mbar_wait_role(FMT == 2 ? &aempty[stage] : &empty[stage], phase ^ 1, chunk & kFxSpinFlag);",
        "\n        FXTR(7, threadIdx.x == 192)")
    ins("        if (lane == 0) mbar_arrive(FMT == 2 ? &afull[stage] : &full[stage]);", "\n        FXTR(8, threadIdx.x == 192)")
    src = src.rstrip()
    assert src.endswith("}  // namespace xpgb")
    src += ('\n\nextern "C" int xpgb_debug_fx_trace(unsigned long long* host) {\n'
            "  return (int)cudaMemcpyFromSymbol(host, xpgb::g_fx_trace, sizeof(unsigned long long) * 10 * 64);\n}\n")
    sys.stdout.write(src)


if __name__ == "__main__":
    main()
