import os, sys
sys.path.insert(0, os.getcwd())
os.environ["SYMCON_KCONFIG"] = "da_s=1"
import torch
from paper_2504_10700_b200.ops import SymmetricContraction
from synth.inputs import CONFIGS, make_config_inputs
cfg = CONFIGS["tiny"]
sc = SymmetricContraction(cfg.lmax_in, cfg.correlation, cfg.out_L, cfg.n_elements, cfg.channels, device=0)
A, W, ne, dB = make_config_inputs(cfg, sc.block_sizes(), sc.out_dim, device="cuda")
B = sc.forward_raw(A, W, ne)
torch.cuda.synchronize()
print("fwd ok")
dA, dW = sc.backward_raw(A, W, ne, dB, need_dW=False)
torch.cuda.synchronize()
print("dA ok")
