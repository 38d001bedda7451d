"""Multi-GPU (>= 2 devices, skipped otherwise): the NVLink peer-memory dW all-reduce
(symcon_peer_allreduce via dist.PeerReducer) against NCCL's all-reduce, and bitwise agreement of
the reduced dW across ranks."""
import os
import socket

import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, algo=1):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    from paper_2504_10700_b200.ops import SymmetricContraction
    from paper_2504_10700_b200.dist import DataParallelContraction
    from synth.inputs import gen_A, gen_W, gen_node_elem, gen_dB
    sc = SymmetricContraction(3, 3, (0, 1), 17, 64, device=rank)
    W = gen_W(17, sc.block_sizes(), 64, "cuda")
    res = []
    for step in range(3):   # several steps: both symmetric buffers and increasing epochs
        N = 3000 + 500 * rank + 100 * step
        A = gen_A(N, 64, 16, "cuda", seed=10 * step + rank)
        ne = gen_node_elem(N, 17, "zipf", "cuda", seed=10 * step + rank)
        dB = gen_dB(N, sc.out_dim, "cuda", seed=10 * step + rank)
        dp = DataParallelContraction(sc, allreduce="peer", peer_algo=algo) if step == 0 else dp
        sc.forward_raw(A, W, ne)
        dA, dW = dp.backward(A, W, ne, dB)
        _, local = sc.backward_raw(A, W, ne, dB, need_dA=False)
        ref = local.clone()
        dist.all_reduce(ref)
        torch.cuda.synchronize()
        dp.check()
        err = (dW - ref).abs().max().item() / ref.abs().max().item()
        allw = [torch.empty_like(dW) for _ in range(world)]
        dist.all_gather(allw, dW)
        same = all(torch.equal(allw[0], x) for x in allw)
        uA = gen_A(N, 64, 16, "cuda", seed=77 + step)
        _, _, Wb = dp.backward2(A, W, ne, dB, uA)
        _, _, Wl = sc.backward2_raw(A, W, ne, dB, uA, False, False, True)
        dist.all_reduce(Wl)
        torch.cuda.synchronize()
        err2 = (Wb - Wl).abs().max().item() / Wl.abs().max().item()
        res.append((max(err, err2), same))
    q.put((rank, res))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("algo", [1, 2])
def test_peer_allreduce_matches_nccl(algo):
    """one-shot and two-shot peer all-reduce on all visible GPUs (2 or 4) against NCCL."""
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q, algo)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    out = [q.get() for _ in range(world)]
    for rank, res in out:
        for err, same in res:
            assert err < 1e-6 and same, (rank, err, same)


def _graph_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    torch.cuda.set_device(rank)
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    from paper_2504_10700_b200.ops import SymmetricContraction
    from paper_2504_10700_b200.dist import DataParallelContraction
    from synth.inputs import gen_A, gen_W, gen_node_elem, gen_dB
    sc = SymmetricContraction(3, 3, (0, 1), 9, 64, device=rank)
    W = gen_W(9, sc.block_sizes(), 64, "cuda")
    ins = []
    for j in range(2):
        N = 2000 + 300 * rank + 50 * j
        ins.append((gen_A(N, 64, 16, "cuda", seed=j + 10 * rank), gen_node_elem(N, 9, "zipf", "cuda", seed=j + 10 * rank),
                    gen_dB(N, sc.out_dim, "cuda", seed=j + 10 * rank)))
    dp = DataParallelContraction(sc, allreduce="peer")
    outs = [torch.empty_like(W) for _ in range(2)]
    dAs = [torch.empty_like(x[0]) for x in ins]
    for j in range(2):                       # eager warm-up (creates the symmetric buffers)
        A, ne, dB = ins[j]
        sc.forward_raw(A, W, ne)
        dp.backward(A, W, ne, dB, dA=dAs[j], dW=outs[j])
    torch.cuda.synchronize()
    graphs = []
    for j in range(2):                       # captured with buffer parities 0 and 1
        g = torch.cuda.CUDAGraph()
        A, ne, dB = ins[j]
        with torch.cuda.graph(g):
            sc.forward_raw(A, W, ne)
            dp.backward(A, W, ne, dB, dA=dAs[j], dW=outs[j])
        graphs.append(g)
    refs = []
    for j in range(2):
        A, ne, dB = ins[j]
        _, loc = sc.backward_raw(A, W, ne, dB, need_dA=False)
        dist.all_reduce(loc)
        refs.append(loc)
    torch.cuda.synchronize()
    errs = []
    for it in range(6):                      # alternate replays: epochs advance on the device
        j = it % 2
        graphs[j].replay()
        torch.cuda.synchronize()
        errs.append((outs[j] - refs[j]).abs().max().item() / refs[j].abs().max().item())
    q.put((rank, max(errs), int(dp._peer.err.item())))   # (error word read after the replays synchronised)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs 2 GPUs")
def test_peer_allreduce_in_cuda_graph_replays():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_graph_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=600)
        assert p.exitcode == 0
    for _ in range(2):
        rank, err, flag = q.get()
        assert err < 1e-6 and flag == 0, (rank, err, flag)
