"""Time kernel-config variants (env SYMCON_KCONFIG) on one workload in a single GPU session.

    python tools/variants.py [--config mp_medium] "" "coef_lookahead=6" "tile_warps=8" ...
Prints one JSON line per variant with per-kernel average ms (libsymcon launch timer).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mp_medium")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--bwd2", action="store_true", help="also run the double backward each iteration")
    ap.add_argument("variants", nargs="*", default=[""])
    args = ap.parse_args()
    import torch
    from paper_2504_10700_b200.ops import SymmetricContraction
    from paper_2504_10700_b200 import _lib
    from synth.inputs import CONFIGS, make_config_inputs
    cfg = CONFIGS[args.config]
    base = None
    for v in args.variants:
        os.environ["SYMCON_KCONFIG"] = "" if v in ("base", '""') else v
        try:
            sc = SymmetricContraction(cfg.lmax_in, cfg.correlation, cfg.out_L, cfg.n_elements, cfg.channels, device=0)
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"variant": v, "error": str(e)[:300]}), flush=True)
            continue
        if base is None:
            base = make_config_inputs(cfg, sc.block_sizes(), sc.out_dim, device="cuda")
        A, W, ne, dB = base
        uA = torch.randn(A.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(5)) if args.bwd2 else None
        ck2 = None
        B = torch.empty((A.shape[0], sc.out_dim), device="cuda")
        dA, dW = torch.empty_like(A), torch.empty_like(W)
        for _ in range(3):
            sc.forward_raw(A, W, ne, B=B)
            sc.backward_raw(A, W, ne, dB, dA=dA, dW=dW, reuse=True)
        torch.cuda.synchronize()
        _lib.symcon_profile_enable(sc.plan, 1)
        _lib.symcon_profile_reset(sc.plan)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sys.path.insert(0, ROOT)
        from bench import ClockSampler
        with ClockSampler(0) as clk:
            clk.start()
            e0.record()
            for _ in range(args.iters):
                sc.forward_raw(A, W, ne, B=B)
                sc.backward_raw(A, W, ne, dB, dA=dA, dW=dW, reuse=True)
                if args.bwd2:
                    ck2 = sc.backward2_raw(A, W, ne, dB, uA, reuse=True)
            e1.record()
            torch.cuda.synchronize()
            clk.end()
        prof = _lib.symcon_profile_read(sc.plan)
        _lib.symcon_profile_enable(sc.plan, 0)
        s, bad = sc.check_device_error()
        out = {"variant": v, "ms_per_step": e0.elapsed_time(e1) / args.iters, "status": s, "clocks": clk.summary(),
               "kernels_ms": {k: round(t / max(n, 1), 4) for k, (n, t) in prof.items()},
               "checksum": [float(B.double().abs().sum()), float(dA.double().abs().sum()), float(dW.double().abs().sum())]
               + ([float(x.double().abs().sum()) for x in ck2] if ck2 else [])}
        print(json.dumps(out), flush=True)
        del sc


if __name__ == "__main__":
    main()
