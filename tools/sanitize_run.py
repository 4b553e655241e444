"""A tiny paged run through every tier for compute-sanitizer (memcheck / racecheck / synccheck):
raw host tier, exponent-Huffman host records, Huffman device tier decoded into the ring, FX4 device
tier read in place by the decode-into-GEMM kernel (with the gate/up -> down overlap), a mixed
FX4 + Huffman device tier, a sub-layer ring, CTA-pair GEMMs, poisoned blocks.  Each run is checked against the resident model.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import numpy as np

    import paper_2604_02715_b200 as X

    spec = X.ModelSpec(2, 8, 256, 512)
    container = X.generate_synthetic_model(spec, 7)
    dev = [X.Backend(1, X.BackendKind.COMPRESSED_DEVICE, 300e9, 1 << 40), X.Backend(2, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    host = [X.Backend(1, X.BackendKind.HOST_OFFLOAD, 30e9, 1 << 40)]
    cases = [
        ("raw host tier", host, None, dict()),
        ("Huffman host records, ring of 4", host, None, dict(host_codec=True, ring_experts=4)),
        ("Huffman device tier into the ring", dev, 0.5, dict(host_codec=True)),
        ("FX4 device tier, decode-into-GEMM", dev, 0.5, dict(host_codec=True, device_format="fx4", fused_decode=True)),
        ("Huffman device tier, decode-into-GEMM", dev, 1.0, dict(fused_decode=True)),
        ("FX4 wholly in place (gate/up->down overlap)", dev, 1.0, dict(device_format="fx4", fused_decode=True)),
        ("mixed FX4 + Huffman device tier (mode 2)", dev, 1.0, dict(mixed=True)),
    ]
    for T in (16, 300):  # decode-sized groups (1-CTA kernels) and CTA-pair groups
        fwd = X.ForwardSpec(T, 2, 7)
        x = np.random.default_rng(T).standard_normal((T, spec.hidden_dim), dtype=np.float32)
        base = X.resident_baseline(1, spec, container, fwd, acts=x.copy())
        for name, backends, alpha, kw in cases:
            hier = X.StorageHierarchy(container, None, X.plan_placement(spec, backends, alpha=alpha), backends)
            kw = dict(kw)
            mixed = kw.pop("mixed", False)
            runner = X.StreamedRunner(spec, hier, fwd, **kw)
            if mixed:
                fmts = np.zeros((spec.num_layers, spec.experts_per_layer, 2), dtype=bool)
                fmts[:, spec.experts_per_layer // 2:, :] = True
                runner.ctx.set_device_formats(fmts)
                runner.ctx.set_fused_decode(2)
            runner.ctx.set_hazard_checks(poison=True)
            rep = runner.run(1, acts=x.copy())
            ok = (rep.page_fault is None and rep.violations == [] and
                  np.asarray(rep.final_activations).tobytes() == np.asarray(base).tobytes())
            print(f"T={T:4d} {name:40s} {'ok' if ok else 'MISMATCH'}", flush=True)
            del runner


if __name__ == "__main__":
    main()
