"""a8 dW all-reduce ("all-reduce") on ONE GPU: the product's peer
all-reduce kernels, their barrier/epoch protocol and their rank-order sums, without several GPUs.

* production launch (symcon_peer_allreduce_ex, gridDim.y = 1), one rank per call, ranks run one
  after another on one stream: the pads of the ranks that have not run yet are pre-signalled, so
  no launch waits on a later one (ranks that wait on each other must never be separate launches
  on one GPU). Covers the one-shot sum order, host and device epochs and buffer alternation.
* emulation (symcon_peer_allreduce_emulate): all ranks' blocks in ONE cooperative launch,
  rank = blockIdx.y, same kernel code: covers the one-shot and the two-shot (reduce-scatter in
  place + grid arrival counter + second barrier + all-gather) for world 2..8 and ragged n.
* the hard timeout: a peer that never arrives -> err = 1, NaN output, symcon_peer_check raises.
Expected values: the fp32 sum in rank order ((b0 + b1) + b2) + ..., computed by torch
elementwise (same rounding, so the comparison is bitwise).
"""
import pytest
import torch

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2504_10700_b200 import _lib


def _bufs(world, n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn(max(n, 1), generator=g, device="cuda")[:n] if n else torch.empty(4, device="cuda")[:0]
            for _ in range(world)]


def _rank_order_sum(bufs):
    s = bufs[0].clone()
    for b in bufs[1:]:
        s += b
    return s


def _st():
    return torch.cuda.current_stream().cuda_stream


@pytest.mark.parametrize("world", [2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 7, 4096, 1_000_003])
def test_one_shot_sequential_ranks_host_and_device_epochs(world, n):
    bufs = [[b.clone() for b in _bufs(world, n, 11 + world)], [b.clone() for b in _bufs(world, n, 23 + world)]]
    pads = [torch.zeros(2 * world + 1, dtype=torch.int32, device="cuda") for _ in range(world)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    counters = [torch.zeros(1, dtype=torch.int32, device="cuda") for _ in range(world)]
    for step, use_dev in enumerate([False, True, False, True]):   # epochs 1..4, both buffers twice
        epoch = step + 1
        bb = bufs[step % 2]
        ref = _rank_order_sum(bb)
        for r in range(world):
            for p in range(r + 1, world):   # ranks p > r "arrived first" at this epoch
                pads[r][p] = epoch
        outs = [torch.full((n,), 7.0, device="cuda") for _ in range(world)]
        for r in range(world):
            if use_dev:
                counters[r].fill_(epoch - 1)   # the device epoch reads counter + 1
                _lib.symcon_peer_allreduce_ex([b.data_ptr() for b in bb], [p.data_ptr() for p in pads], r, n, 0,
                                              counters[r].data_ptr(), 1, 1 << 16, outs[r].data_ptr(), err.data_ptr(), _st())
            else:
                _lib.symcon_peer_allreduce_ex([b.data_ptr() for b in bb], [p.data_ptr() for p in pads], r, n, epoch,
                                              None, 1, 1 << 16, outs[r].data_ptr(), err.data_ptr(), _st())
        _lib.symcon_peer_check(err.data_ptr(), _st())
        for r in range(world):
            assert torch.equal(outs[r], ref), (world, n, step, r)
            if use_dev:
                assert int(counters[r].item()) == epoch       # bumped once per call
        for r in range(world):
            assert all(int(v) == epoch for v in pads[r][:world].tolist())


@pytest.mark.parametrize("algo", [1, 2])
@pytest.mark.parametrize("world", [2, 3, 4, 5, 8])
@pytest.mark.parametrize("n", [1, 5, 8, 1023, 262_147, 979_456])
def test_emulated_ranks_one_and_two_shot(algo, world, n):
    bufs = _bufs(world, n, 100 * world + n % 97)
    orig = [b.clone() for b in bufs]
    ref = _rank_order_sum(orig)
    pads = [torch.zeros(2 * world + 1, dtype=torch.int32, device="cuda") for _ in range(world)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for epoch in (1, 2, 3):   # repeated calls: increasing epochs, the grid counter reset each time
        for r in range(world):
            bufs[r].copy_(orig[r])   # the two-shot reduces slice r in place into bufs[r]
        outs = [torch.full((n,), 3.0, device="cuda") for _ in range(world)]
        _lib.symcon_peer_allreduce_emulate([b.data_ptr() for b in bufs], [p.data_ptr() for p in pads],
                                           [o.data_ptr() for o in outs], n, epoch, algo, 1 << 18, err.data_ptr(), _st())
        _lib.symcon_peer_check(err.data_ptr(), _st())
        for r in range(world):
            assert torch.equal(outs[r], ref), (algo, world, n, epoch, r)
        for r in range(world):
            assert int(pads[r][2 * world].item()) == 0            # grid arrival counter reset
            assert all(int(v) == epoch for v in pads[r][:world].tolist())
            if algo == 2:
                assert all(int(v) == epoch for v in pads[r][world:2 * world].tolist())
        if algo == 1:
            for r in range(world):
                assert torch.equal(bufs[r], orig[r])              # one-shot leaves the partials alone


@pytest.mark.parametrize("algo", [1, 2])
def test_timeout_is_a_hard_error_not_partial_sums(algo):
    world, n = 2, 10_000
    bufs = _bufs(world, n, 5)
    pads = [torch.zeros(2 * world + 1, dtype=torch.int32, device="cuda") for _ in range(world)]
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.zeros(n, device="cuda")
    # rank 1 never arrives; a short spin limit (~1e4 polls of ~200 ns)
    _lib.symcon_peer_allreduce_ex([b.data_ptr() for b in bufs], [p.data_ptr() for p in pads], 0, n, 1, None, algo,
                                  10_000, out.data_ptr(), err.data_ptr(), _st())
    with pytest.raises(_lib.SymconError) as ei:
        _lib.symcon_peer_check(err.data_ptr(), _st())
    assert ei.value.status == _lib.SYMCON_ETIMEOUT
    assert int(err.item()) == 1
    assert torch.isnan(out).all()


def test_argument_validation():
    b = torch.zeros(8, device="cuda")
    p = torch.zeros(8, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    with pytest.raises(_lib.SymconError):   # misaligned output
        _lib.symcon_peer_allreduce_ex([b.data_ptr()] * 2, [p.data_ptr()] * 2, 0, 4, 1, None, 1, 0, b.data_ptr() + 4,
                                      err.data_ptr(), _st())
    with pytest.raises(_lib.SymconError):   # bad algo
        _lib.symcon_peer_allreduce_ex([b.data_ptr()] * 2, [p.data_ptr()] * 2, 0, 4, 1, None, 3, 0, b.data_ptr(),
                                      err.data_ptr(), _st())
