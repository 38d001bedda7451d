"""ORACLE — test infrastructure only. NOT part of the product.

A plain, slow, obviously-correct fp64 CPU implementation of MACE's symmetric
tensor contraction (Alg. 3; Eq. (2)) and of
the paper's load balancer (Alg. 1), written from the paper
and DESIGN.md's readings before any kernel.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import, call, link or execute anything under
`oracle/`. The CUDA product path (`paper_2504_10700_b200/`) never imports it,
shares no code, headers, tables or constant generators with it, and fails
loudly when its own CUDA library is missing.

Modules:
  so3          real spherical harmonics, complex->real basis, Racah CG,
               real CG with the DESIGN.md sign rule, Wigner-D fitted from SH.
  paths        left-nested coupling paths and their generalized CG tensors U.
  contraction  forward / backward (dA, dW) of Alg. 3, sparse raw-tuple loop,
               and a dense brute-force evaluator for tiny inputs.
  packing      Alg. 1 Create-Balanced-Batches and the Eq. (1)-(5) metrics.
  ceval        ctypes wrapper around oracle/csrc/oracle_eval.c, a plain C
               fp64 OpenMP loop over the same raw tuples (timing + big parity).
  tp           channelwise tensor product (Alg. 2) + edge->node
               sum pooling (Eq. (1)); forward, backward (dY, dh, dR), brute force.

Parity-unpinned functions: none in so3/paths/contraction/packing/tp (see
tests/test_oracle_*.py for each pin). Agreement with MACE/e3nn numeric tables
is unpinned (no e3nn or MACE weights in this environment).
"""
