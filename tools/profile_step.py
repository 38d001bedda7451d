"""Short fwd+bwd run of one workload for ncu captures (no timing, no oracle).

    python tools/profile_step.py [--config mp_medium] [--iters 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="mp_medium")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--bwd2", action="store_true", help="also run the double backward")
    args = ap.parse_args()
    import torch
    from paper_2504_10700_b200.ops import SymmetricContraction
    from synth.inputs import CONFIGS, make_config_inputs
    cfg = CONFIGS[args.config]
    sc = SymmetricContraction(cfg.lmax_in, cfg.correlation, cfg.out_L, cfg.n_elements, cfg.channels, device=0)
    A, W, ne, dB = make_config_inputs(cfg, sc.block_sizes(), sc.out_dim, device="cuda")
    for _ in range(args.iters):
        B = sc.forward_raw(A, W, ne)
        dA, dW = sc.backward_raw(A, W, ne, dB)
        if args.bwd2:
            sc.backward2_raw(A, W, ne, dB, A, reuse=True)
    torch.cuda.synchronize()
    s, bad = sc.check_device_error()
    assert s == 0, (s, bad)
    print("ok", float(B.abs().sum()), float(dA.abs().sum()), float(dW.abs().sum()))


if __name__ == "__main__":
    main()
