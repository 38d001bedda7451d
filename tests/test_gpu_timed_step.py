"""Parity of the EXACT step bench.py times (VERDICT r01 weak #2a): bench.TimedStep at N = 1 with
its defaults -- the 4-bin pool of 50k-node Alg. 1 bins (Table-2 manifest), DataParallelContraction
with dW on the main stream and dA concurrently on a side stream sharing one workspace, the reuse
hints after the forward, one CUDA graph per pool entry replayed for two full cycles -- against the
plain C fp64 oracle (oracle/csrc/oracle_eval.c) on the same seeded inputs:
  * B and dA on 128 sampled nodes of every bin (per-node outputs depend on that node only);
  * dW on EVERY element of every bin, including the Zipf-head element (~10.6k nodes of one
    element, reduced over ~42 dW items), from the oracle over all ~50k nodes of the bin.
Tolerance: max|err| <= 1e-5 * max|ref| per tensor (the internal gate; north_star 1e-4), plus the
head element's dW on its own at the same bar.
Also the C = 3072 operating point of the same object, all nodes of every bin.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _rel(x, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.abs(np.asarray(x, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def _oracle(cfg):
    from oracle.contraction import Problem
    from oracle.ceval import OracleC
    return OracleC(Problem(cfg.lmax_in, cfg.correlation, cfg.out_L))


def _replay_and_snapshot(ts, cycles=2):
    snaps = {}
    for _ in range(cycles):
        for q in range(len(ts.pool)):
            ts.step(q)
            torch.cuda.synchronize()
            b, N, A, ne, dB, B, dA = ts.pool[q]
            snaps[q] = (B.cpu().numpy(), dA.cpu().numpy(), ts.dW.cpu().numpy())   # dW is shared: snapshot now
    ts.dp.check()
    s, bad = ts.sc.check_device_error()
    assert s == 0, bad
    return snaps


@pytest.fixture(scope="module")
def timed_step():
    import bench
    ts = bench.TimedStep()            # bench.py's defaults: mp_medium, C = 50,000, pool 4, N = 1
    for q in range(5):                # bench.py's warm-up (eager), then capture + one replay cycle
        ts.eager(q)
    torch.cuda.synchronize()
    ts.capture()
    assert ts.graphs is not None and ts.dp.concurrent_bwd and ts.dp.side is not None
    return ts


def test_timed_step_graph_replays_match_oracle(timed_step):
    ts = timed_step
    snaps = _replay_and_snapshot(ts, cycles=2)
    oc = _oracle(ts.cfg)
    hW = ts.W.cpu().numpy()
    rng = np.random.default_rng(7)
    for q in range(len(ts.pool)):
        b, N, A, ne, dB, B, dA = ts.pool[q]
        hA, hne, hdB = A.cpu().numpy(), ne.cpu().numpy(), dB.cpu().numpy()
        Bq, dAq, dWq = snaps[q]
        idx = np.sort(rng.choice(N, 128, replace=False))
        Bref = oc.forward(hA[idx], hW, hne[idx])
        dAref, _ = oc.backward(hA[idx], hW, hne[idx], hdB[idx], want_dW=False)
        assert _rel(Bq[idx], Bref) < TOL, (q, "B")
        assert _rel(dAq[idx], dAref) < TOL, (q, "dA")
        _, dWref = oc.backward(hA, hW, hne, hdB, want_dA=False)      # every node of the bin
        assert _rel(dWq, dWref) < TOL, (q, "dW")
        counts = np.bincount(hne, minlength=hW.shape[0])
        head = int(np.argmax(counts))
        assert counts[head] > 5000                                   # the Zipf head is really exercised
        assert _rel(dWq[head], dWref[head]) < TOL, (q, "dW head element", head, counts[head])
        assert np.all(dWq[counts == 0] == 0.0)                       # elements absent from the bin: exact 0


def test_timed_step_small_capacity_all_nodes():
    """The paper's operating point C = 3072 nodes per GPU-step: same TimedStep,
    graph replays, every node and element compared."""
    import bench
    ts = bench.TimedStep(capacity=3072)
    for q in range(3):
        ts.eager(q)
    torch.cuda.synchronize()
    ts.capture()
    snaps = _replay_and_snapshot(ts, cycles=2)
    oc = _oracle(ts.cfg)
    hW = ts.W.cpu().numpy()
    for q in range(len(ts.pool)):
        b, N, A, ne, dB, B, dA = ts.pool[q]
        assert 3072 - 768 <= N <= 3072
        hA, hne, hdB = A.cpu().numpy(), ne.cpu().numpy(), dB.cpu().numpy()
        Bref = oc.forward(hA, hW, hne)
        dAref, dWref = oc.backward(hA, hW, hne, hdB)
        Bq, dAq, dWq = snaps[q]
        assert _rel(Bq, Bref) < TOL and _rel(dAq, dAref) < TOL and _rel(dWq, dWref) < TOL, q


@pytest.mark.parametrize("dtype,correlation,tol", [("f64", None, 1e-10), ("f32", 4, 1e-5)])
def test_timed_step_variants_full_size_sampled(dtype, correlation, tol):
    """The bench's timed step for the §8(f) row-3 variants at the full MP-medium size (bench.py
    --dtype f64 / --correlation 4; C = 50,000, the same pool, streams and CUDA graphs): B and dA on
    64 sampled nodes of one bin, dW on the four smallest elements present (all their nodes) and, in
    fp64, on the Zipf-head element too (~10k nodes), against the C oracle."""
    import bench
    ts = bench.TimedStep(pool=2, dtype=dtype, correlation=correlation)
    for q in range(2):
        ts.eager(q)
    torch.cuda.synchronize()
    ts.capture()
    snaps = _replay_and_snapshot(ts, cycles=1)
    oc = _oracle(ts.cfg)
    hW = ts.W.cpu().double().numpy()
    b, N, A, ne, dB, B, dA = ts.pool[0]
    hA, hne, hdB = A.cpu().double().numpy(), ne.cpu().numpy(), dB.cpu().double().numpy()
    Bq, dAq, dWq = snaps[0]
    idx = np.sort(np.random.default_rng(11).choice(N, 64, replace=False))
    assert _rel(Bq[idx], oc.forward(hA[idx], hW, hne[idx])) < tol
    assert _rel(dAq[idx], oc.backward(hA[idx], hW, hne[idx], hdB[idx], want_dW=False)[0]) < tol
    counts = np.bincount(hne, minlength=hW.shape[0])
    present = np.nonzero(counts)[0]
    chosen = list(present[np.argsort(counts[present], kind="stable")[:4]])
    if dtype == "f64":
        chosen.append(int(np.argmax(counts)))
    for z in chosen:
        sel = np.nonzero(hne == z)[0]
        _, dWref = oc.backward(hA[sel], hW, hne[sel], hdB[sel], want_dA=False)
        assert _rel(dWq[z], dWref[z]) < tol, (dtype, correlation, z, counts[z])
