"""Data-parallel sharding of the contraction over bin-packed molecular graphs.

* BinPackedShards: Alg. 1 (C++ partitioner in libsymcon) over the epoch's
  graph sizes with capacity C and G = world size; bin j runs on rank j % G at step j // G
  (reading s18). Every rank computes the same plan (deterministic, stable sorts,
  PAPER.md:477), so no plan broadcast is needed.
* DataParallelContraction: one training step of the contraction on this rank's bin: forward,
  backward dW, NCCL all-reduce of dW (the one cross-GPU exchange; PAPER.md:960 DDP all-reduce)
  on a communication stream, overlapped with the backward dA kernel. For force training the
  double backward's W_bar is all-reduced the same way, overlapped with its tile kernel.
* allreduce="peer" (default for N > 1 when torch symmetric memory is available): dW is written
  straight into a symmetric (peer-mapped) buffer and libsymcon's own kernel does the cross-GPU
  barrier and the rank-ordered sum over NVLink P2P loads (symcon_peer_allreduce): no NCCL kernel
  competing with the persistent dA grid, bitwise-identical dW on every rank.
"""
import numpy as np
import torch
import torch.distributed as dist

from . import _lib


class BinPackedShards:
    def __init__(self, sizes, capacity, world, rank):
        self.sizes = np.ascontiguousarray(sizes, dtype=np.int64)
        self.capacity, self.world, self.rank = int(capacity), int(world), int(rank)
        self.offsets, self.ids = _lib.symcon_pack_balanced(self.sizes, self.capacity, self.world)
        self.n_bins = len(self.offsets) - 1
        assert self.n_bins % self.world == 0
        self.n_steps = self.n_bins // self.world

    def bin_of(self, step, rank=None):
        return step * self.world + (self.rank if rank is None else rank)

    def graphs(self, step, rank=None):
        b = self.bin_of(step, rank)
        return self.ids[self.offsets[b]:self.offsets[b + 1]]

    def nodes(self, step, rank=None):
        return int(self.sizes[self.graphs(step, rank)].sum())

    def step_imbalance(self, step):
        """max / mean nodes over ranks at one step (1.0 = perfect balance)."""
        loads = np.array([self.nodes(step, r) for r in range(self.world)], dtype=np.float64)
        return float(loads.max() / max(loads.mean(), 1.0))

    def bin_loads(self):
        return np.add.reduceat(self.sizes[self.ids], self.offsets[:-1]) if self.n_bins else np.zeros(0)


class PeerReducer:
    """Two symmetric (peer-mapped) fp32 buffers used alternately per step + one signal pad; the
    all-reduce itself is libsymcon's kernel (no NCCL). algo: 0 auto (two-shot for world >= 8),
    1 one-shot, 2 two-shot (symcon_peer_allreduce_ex). A barrier timeout is a hard error: the
    kernel writes NaN and sets `err`; `check()` raises it (SYMCON_ETIMEOUT)."""

    def __init__(self, numel, device, group=None, algo=0, spin_limit=0):
        import torch.distributed._symmetric_memory as symm
        grp = group if group is not None else dist.group.WORLD
        self.numel = int(numel)
        self.algo, self.spin_limit = int(algo), int(spin_limit)
        self.bufs = [symm.empty(self.numel, dtype=torch.float32, device=device) for _ in range(2)]
        self.hdl = [symm.rendezvous(b, grp) for b in self.bufs]
        self.rank, self.world = self.hdl[0].rank, self.hdl[0].world_size
        # slots [0, world): first barrier, [world, 2 world): two-shot second barrier, 2 world: grid counter
        pad = self.hdl[0].get_signal_pad(self.rank, (2 * self.world + 1,), dtype=torch.int32)
        pad.zero_()
        self.err = torch.zeros(1, dtype=torch.int32, device=device)
        self.counter = torch.zeros(1, dtype=torch.int32, device=device)   # device epoch (graph-capturable)
        torch.cuda.synchronize(device)
        dist.barrier(group=group)
        self.parity = 0

    def buffer(self):
        return self.bufs[self.parity]

    def allreduce(self, out, stream):
        """Epoch kept on the device, so the call can be captured in a CUDA graph; the buffer parity
        alternates per call (capture an even number of steps)."""
        h = self.hdl[self.parity]
        _lib.symcon_peer_allreduce_ex(list(h.buffer_ptrs), list(self.hdl[0].signal_pad_ptrs), self.rank, self.numel, 0,
                                      self.counter.data_ptr(), self.algo, self.spin_limit, out.data_ptr(),
                                      self.err.data_ptr(), stream)
        self.parity ^= 1
        return out

    def check(self):
        """Synchronises; raises SymconError (SYMCON_ETIMEOUT) if a barrier of an earlier call timed out."""
        _lib.symcon_peer_check(self.err.data_ptr(), torch.cuda.current_stream(self.err.device).cuda_stream)


class DataParallelContraction:
    """Forward + backward of one rank's bin. The dW kernels run on the main stream and the dA
    kernel on a side stream (concurrently; `concurrent_bwd`), and for N > 1 the dW all-reduce
    runs on a communication stream as soon as dW is ready, overlapped with dA."""

    def __init__(self, sc, group=None, overlap=True, concurrent_bwd=None, allreduce=None, peer_algo=0):
        self.sc = sc
        self.group = group
        self.overlap = overlap
        self.allreduce = allreduce or "peer"
        self.peer_algo = int(peer_algo)
        self._peer = None
        self._peer2 = None
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        # measured: dA concurrent with dW helps with <= 4 output slots per channel (MP-medium 1.08 vs
        # 1.12 ms/step; the dW all-reduce then runs as SMs free up); at 9 slots (large) the 3-CTA-per-item
        # dW_r and the persistent dA slow each other down (21.6 vs 18.2 ms), so dA follows dW there
        out_slots = sc.out_dim // max(sc.channels, 1)
        self.concurrent_bwd = (out_slots <= 4) if concurrent_bwd is None else concurrent_bwd
        self.side = torch.cuda.Stream(device=sc.device) if self.concurrent_bwd else None
        self.comm = torch.cuda.Stream(device=sc.device) if self.world > 1 else None
        self.launches = 0

    def check(self):
        """Synchronises; raises if a peer all-reduce barrier of an earlier step timed out (the
        kernel then wrote NaN into dW / W_bar instead of partial sums)."""
        for r in (self._peer, getattr(self, "_peer2", None)):
            if r is not None:
                r.check()

    def forward(self, A, W, node_elem, B=None):
        B = self.sc.forward_raw(A, W, node_elem, B=B)
        self.launches += self.sc.last_launch_count()
        return B

    def backward(self, A, W, node_elem, dB, dA=None, dW=None):
        sc = self.sc
        if self.world == 1 and not self.concurrent_bwd:
            dA, dW = sc.backward_raw(A, W, node_elem, dB, dA=dA, dW=dW, reuse=True)
            self.launches += sc.last_launch_count()
            return dA, dW
        if self.world == 1:
            # dW and dA kernels on two streams (they can share SMs as either drains)
            main = torch.cuda.current_stream(sc.device)
            self.side.wait_stream(main)          # inputs ready; dW and dA then run concurrently
            _, dW = sc.backward_raw(A, W, node_elem, dB, need_dA=False, dW=dW, reuse=True)
            self.launches += sc.last_launch_count()
            with torch.cuda.stream(self.side):
                dA, _ = sc.backward_raw(A, W, node_elem, dB, need_dW=False, dA=dA, reuse=True, ws_key="default")
                self.launches += sc.last_launch_count()
            main.wait_stream(self.side)
            return dA, dW
        main = torch.cuda.current_stream(sc.device)
        if self.allreduce == "peer" and self._peer is None:
            try:
                self._peer = PeerReducer(W.numel(), sc.device, self.group, algo=self.peer_algo)
            except Exception as exc:  # noqa: BLE001  (no symmetric memory on this system: NCCL)
                import sys
                print(f"[symcon] peer-memory all-reduce unavailable ({exc!r}); using NCCL", file=sys.stderr)
                self.allreduce = "nccl"
        if self.allreduce == "peer":
            if dW is None:
                dW = torch.empty_like(W)
            if self.side is not None:
                self.side.wait_stream(main)
            part = self._peer.buffer()[:W.numel()].view(W.shape)
            sc.backward_raw(A, W, node_elem, dB, need_dA=False, dW=part, reuse=True)
            self.launches += sc.last_launch_count()
            if self.side is not None:
                with torch.cuda.stream(self.side):
                    dA, _ = sc.backward_raw(A, W, node_elem, dB, need_dW=False, dA=dA, reuse=True)
                    self.launches += sc.last_launch_count()
            self._peer.allreduce(dW, main.cuda_stream)
            self.launches += 2
            if self.side is not None:
                main.wait_stream(self.side)
            else:
                dA, _ = sc.backward_raw(A, W, node_elem, dB, need_dW=False, dA=dA, reuse=True)
                self.launches += sc.last_launch_count()
            return dA, dW
        if not self.overlap:
            dA, dW = sc.backward_raw(A, W, node_elem, dB, dA=dA, dW=dW, reuse=True)
            self.launches += sc.last_launch_count()
            dist.all_reduce(dW, group=self.group)
            return dA, dW
        # dW first (bucketing and W-fold reused from the forward), its all-reduce on the comm stream;
        # dA on a side stream from the start (concurrent with dW and with the all-reduce)
        if self.concurrent_bwd:
            self.side.wait_stream(main)
        _, dW = sc.backward_raw(A, W, node_elem, dB, need_dA=False, dW=dW, reuse=True)
        self.launches += sc.last_launch_count()
        ev = torch.cuda.Event()
        ev.record(main)
        self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            dist.all_reduce(dW, group=self.group)
        dW.record_stream(self.comm)
        if self.concurrent_bwd:
            with torch.cuda.stream(self.side):
                dA, _ = sc.backward_raw(A, W, node_elem, dB, need_dW=False, dA=dA, reuse=True)
                self.launches += sc.last_launch_count()
            main.wait_stream(self.side)
        else:
            dA, _ = sc.backward_raw(A, W, node_elem, dB, need_dW=False, dA=dA, reuse=True)
            self.launches += sc.last_launch_count()
        main.wait_stream(self.comm)
        return dA, dW

    def backward2(self, A, W, node_elem, dB, uA, need_dB=True, need_A=True):
        """Double backward of this rank's bin (force loss): W_bar first (all-reduced over ranks on
        the communication stream), then dB_bar / A_bar, which stay local to the rank's nodes."""
        sc = self.sc
        if self.world == 1:
            out = sc.backward2_raw(A, W, node_elem, dB, uA, need_dB, need_A, True, reuse=True)
            self.launches += sc.last_launch_count()
            return out
        main = torch.cuda.current_stream(sc.device)
        if self.allreduce == "peer" and self._peer2 is None:
            try:
                self._peer2 = PeerReducer(W.numel(), sc.device, self.group, algo=self.peer_algo)
            except Exception as exc:  # noqa: BLE001
                import sys
                print(f"[symcon] peer-memory all-reduce unavailable ({exc!r}); using NCCL", file=sys.stderr)
                self.allreduce = "nccl"
        if self.allreduce == "peer":
            part = self._peer2.buffer()[:W.numel()].view(W.shape)
            side = self.side if self.side is not None else main
            if side is not main:
                side.wait_stream(main)
            # W_bar partial straight into the symmetric buffer (main), the tile part on the side stream
            sc.backward2_raw(A, W, node_elem, dB, uA, False, False, True, reuse=True, W_bar=part)
            self.launches += sc.last_launch_count()
            dBb = Ab = None
            if need_dB or need_A:
                with torch.cuda.stream(side):
                    dBb, Ab, _ = sc.backward2_raw(A, W, node_elem, dB, uA, need_dB, need_A, False, reuse=True)
                    self.launches += sc.last_launch_count()
            Wb = torch.empty_like(W)
            self._peer2.allreduce(Wb, main.cuda_stream)
            self.launches += 2
            if side is not main:
                main.wait_stream(side)
            return dBb, Ab, Wb
        _, _, Wb = sc.backward2_raw(A, W, node_elem, dB, uA, False, False, True, reuse=True)
        self.launches += sc.last_launch_count()
        self.comm.wait_stream(main)
        with torch.cuda.stream(self.comm):
            dist.all_reduce(Wb, group=self.group)
        Wb.record_stream(self.comm)
        dBb = Ab = None
        if need_dB or need_A:
            dBb, Ab, _ = sc.backward2_raw(A, W, node_elem, dB, uA, need_dB, need_A, False, reuse=True)
            self.launches += sc.last_launch_count()
        main.wait_stream(self.comm)
        return dBb, Ab, Wb
