"""Determinism probe of the decode-into-GEMM kernel: the same paged stack run several times with
FX4 fused, compared with the resident model layer by layer."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np
    import torch

    import paper_2604_02715_b200 as X
    from paper_2604_02715_b200.exponent_codec import CompressedModel

    N, L, H, F, k = 2, 8, 4096, 14336, 2
    T = int(os.environ.get("T", "256"))
    spec = X.ModelSpec(N, L, H, F)
    fwd = X.ForwardSpec(T, k, 7)
    container = X.generate_fast_model(spec, 7)
    backends = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 50),
                X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 50)]
    hier = X.StorageHierarchy(container, CompressedModel.from_container(container),
                              X.plan_placement(spec, backends, alpha=1.0), backends)
    x = torch.from_numpy(np.random.default_rng(3).standard_normal((T, H), dtype=np.float32)).cuda()
    model = X.ResidentModel(spec, container, max_tokens=T)
    y, _ = model.run(1, fwd, x.clone())
    ref = y.cpu().numpy()
    del model
    for fmt, fused in (("fx4", True), ("fx4", False), ("huffman", True)):
        runner = X.StreamedRunner(spec, hier, fwd, fused_decode=fused, device_format=fmt)
        for rep_i in range(4):
            rep = runner.run(1, acts=x.clone())
            out = rep.final_activations.cpu().numpy()
            bad = np.argwhere(out != ref)
            rows = sorted(set(int(r) for r, _ in bad))[:10]
            cols = sorted(set(int(c) for _, c in bad))
            print(json.dumps({"fmt": fmt, "fused": fused, "rep": rep_i, "mismatches": int(len(bad)),
                              "rows": rows, "n_cols": len(cols), "cols_head": cols[:12],
                              "max_rel": float(np.max(np.abs(out - ref)) / (np.max(np.abs(ref)) + 1e-30))}), flush=True)
        del runner
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
