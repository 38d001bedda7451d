"""PyTorch glue for libsymcon: device memory, streams and autograd. No compute here.

    sc = SymmetricContraction(lmax_in=3, correlation=3, out_L=(0, 1), num_elements=89,
                              channels=128, device=0)
    B = sc(A, W, node_elem)          # autograd-aware; backward gives dA and dW, and with
                                     # create_graph=True the backward is differentiable again
                                     # (double backward for force training, symcon_backward2)

Every numeric step (bucketing, W-fold, forward, dA, dW, reductions) runs in the CUDA
kernels of libsymcon.so through the C ABI; tensors only provide pointers.
"""
import torch

from . import _lib


def _stream_ptr(device):
    return torch.cuda.current_stream(device).cuda_stream


class SymmetricContraction:
    """One plan (U tables + loaded sm_100a kernels) per (config, device)."""

    def __init__(self, lmax_in, correlation, out_L, num_elements, channels, device=None, dtype=torch.float32):
        if not torch.cuda.is_available():
            raise RuntimeError("SymmetricContraction needs a CUDA device (libsymcon has no CPU path)")
        if dtype not in (torch.float32, torch.float64):
            raise ValueError("dtype must be torch.float32 or torch.float64")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.lmax_in, self.correlation, self.out_L = lmax_in, correlation, tuple(out_L)
        self.num_elements, self.channels = num_elements, channels
        self.dtype = dtype
        code = _lib.SYMCON_F64 if dtype == torch.float64 else _lib.SYMCON_F32
        with torch.cuda.device(self.device):
            self.plan = _lib.symcon_build_tables_ex(lmax_in, correlation, list(out_L), num_elements, channels,
                                                    self.device.index, code)
        info = _lib.symcon_plan_info(self.plan)
        self.info = info
        self.n_paths = info.n_paths
        self.n_lm = (lmax_in + 1) ** 2
        self.out_dim = info.out_dim
        self._ws = {}

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan is not None:
            _lib.symcon_destroy(plan)
            self.plan = None

    # ------------------------------------------------------------------ helpers
    def block_sizes(self):
        """[(L, nu, n_eta)] in W column order."""
        out = []
        for L in range(self.info.n_out):
            for nu in range(self.correlation):
                n = self.info.eta[L][nu]
                if n:
                    out.append((self.info.out_L[L], nu + 1, n))
        return out

    def workspace(self, num_nodes, key="default"):
        nbytes = _lib.symcon_workspace_bytes(self.plan, num_nodes)
        ws = self._ws.get(key)
        if ws is None or ws.numel() < nbytes:
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[key] = ws
        return ws

    def _check(self, A, W, node_elem):
        N = A.shape[0]
        assert A.is_cuda and A.device == self.device and A.dtype == self.dtype and A.is_contiguous()
        assert A.shape == (N, self.channels, self.n_lm), A.shape
        assert W.dtype == self.dtype and W.is_contiguous() and W.shape == (self.num_elements, self.n_paths, self.channels)
        assert node_elem.dtype == torch.int32 and node_elem.is_contiguous() and node_elem.shape == (N,)
        return N

    # ------------------------------------------------------------------ raw calls
    def forward_raw(self, A, W, node_elem, B=None, ws_key="default"):
        N = self._check(A, W, node_elem)
        if B is None:
            B = torch.empty((N, self.out_dim), dtype=self.dtype, device=self.device)
        ws = self.workspace(N, ws_key)
        fn = _lib.symcon_forward_f64 if self.dtype == torch.float64 else _lib.symcon_forward
        fn(self.plan, N, A.data_ptr(), W.data_ptr(), node_elem.data_ptr(), B.data_ptr(),
           ws.data_ptr(), ws.numel(), _stream_ptr(self.device))
        return B

    def backward_raw(self, A, W, node_elem, dB, need_dA=True, need_dW=True, dA=None, dW=None, ws_key="default",
                     reuse=False):
        """reuse=True passes SYMCON_REUSE_BUCKETS|FOLD: the bucketing and W-fold left in the
        workspace by the preceding forward (same node_elem / W tensors) are reused."""
        N = self._check(A, W, node_elem)
        assert dB.dtype == self.dtype and dB.is_contiguous() and dB.shape == (N, self.out_dim)
        if need_dA and dA is None:
            dA = torch.empty_like(A)
        if need_dW and dW is None:
            dW = torch.empty_like(W)
        ws = self.workspace(N, ws_key)
        flags = (_lib.SYMCON_REUSE_BUCKETS | _lib.SYMCON_REUSE_FOLD) if reuse else 0
        fn = _lib.symcon_backward_f64 if self.dtype == torch.float64 else _lib.symcon_backward_ex
        fn(self.plan, N, A.data_ptr(), W.data_ptr(), node_elem.data_ptr(), dB.data_ptr(),
           dA.data_ptr() if need_dA else None, dW.data_ptr() if need_dW else None,
           ws.data_ptr(), ws.numel(), flags, _stream_ptr(self.device))
        return (dA if need_dA else None), (dW if need_dW else None)

    def backward2_raw(self, A, W, node_elem, dB, uA, need_dB=True, need_A=True, need_W=True, ws_key="default",
                      reuse=False, W_bar=None, uW=None):
        """Double backward: (dB_bar, A_bar, W_bar) = derivatives of <uA, dA(A, W, dB)> + <uW, dW(A, dB)>
        (symcon_backward2_ex; uA or uW may be None). W_bar may be given (e.g. a symmetric buffer for the
        peer all-reduce)."""
        N = self._check(A, W, node_elem)
        assert dB.dtype == torch.float32 and dB.is_contiguous() and dB.shape == (N, self.out_dim)
        assert uA is not None or uW is not None
        if uA is not None:
            assert uA.dtype == torch.float32 and uA.is_contiguous() and uA.shape == A.shape
        if uW is not None:
            assert uW.dtype == torch.float32 and uW.is_contiguous() and uW.shape == W.shape
        dBb = torch.empty_like(dB) if need_dB else None
        Ab = torch.empty_like(A) if need_A else None
        Wb = (W_bar if W_bar is not None else torch.empty_like(W)) if need_W else None
        ws = self.workspace(N, ws_key)
        flags = (_lib.SYMCON_REUSE_BUCKETS | _lib.SYMCON_REUSE_FOLD) if reuse else 0
        ptr = lambda x: x.data_ptr() if x is not None else None
        _lib.symcon_backward2_ex(self.plan, N, A.data_ptr(), W.data_ptr(), node_elem.data_ptr(), dB.data_ptr(),
                                 ptr(uA), ptr(uW), ptr(dBb), ptr(Ab), ptr(Wb), ws.data_ptr(), ws.numel(), flags,
                                 _stream_ptr(self.device))
        return dBb, Ab, Wb

    def check_device_error(self, ws_key="default"):
        ws = self._ws.get(ws_key)
        if ws is None:
            return 0, -1
        return _lib.symcon_check_device_error(self.plan, ws.data_ptr(), _stream_ptr(self.device))

    def last_launch_count(self):
        return _lib.symcon_last_launch_count(self.plan)

    # ------------------------------------------------------------------ autograd
    def __call__(self, A, W, node_elem):
        return _SymconFn.apply(A, W, node_elem, self)


class _SymconFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, A, W, node_elem, sc):
        ctx.sc = sc
        A, W, node_elem = A.contiguous(), W.contiguous(), node_elem.contiguous()
        ctx.save_for_backward(A, W, node_elem)   # the contiguous tensors the kernels ran on
        return sc.forward_raw(A, W, node_elem)

    @staticmethod
    def backward(ctx, dB):
        A, W, node_elem = ctx.saved_tensors
        if torch.is_grad_enabled():
            # create_graph=True (training on forces): the backward is itself differentiable
            dA, dW = _SymconBwdFn.apply(A, W, node_elem, dB, ctx.sc)
            return dA, dW, None, None
        dA, dW = ctx.sc.backward_raw(A, W, node_elem, dB.contiguous(), ctx.needs_input_grad[0], ctx.needs_input_grad[1],
                                     reuse=True)
        return dA, dW, None, None


class _SymconBwdFn(torch.autograd.Function):
    """(A, W, dB) -> (dA, dW) with its own backward: the uA terms (symcon_backward2 kernels) and the uW
    terms (dB_bar += B(A, uW), A_bar += dA(A, uW, dB)) in one symcon_backward2_ex call."""

    @staticmethod
    def forward(ctx, A, W, node_elem, dB, sc):
        ctx.sc = sc
        A, W, node_elem, dB = A.contiguous(), W.contiguous(), node_elem.contiguous(), dB.contiguous()
        ctx.save_for_backward(A, W, node_elem, dB)
        return sc.backward_raw(A, W, node_elem, dB)

    @staticmethod
    @torch.autograd.function.once_differentiable
    def backward(ctx, uA, uW):
        A, W, node_elem, dB = ctx.saved_tensors
        sc = ctx.sc
        need_A, need_W, need_dB = ctx.needs_input_grad[0], ctx.needs_input_grad[1], ctx.needs_input_grad[3]
        uA = uA.contiguous() if uA is not None else None
        uW = uW.contiguous() if uW is not None else None
        need_W = need_W and uA is not None          # W_bar has no uW term (dW does not depend on W)
        if (uA is None and uW is None) or not (need_A or need_W or need_dB):
            return None, None, None, None, None
        # uA and uW terms are summed inside libsymcon (symcon_backward2_ex): no arithmetic here
        dB_bar, A_bar, W_bar = sc.backward2_raw(A, W, node_elem, dB, uA, need_dB, need_A, need_W, uW=uW)
        return A_bar, W_bar, None, dB_bar, None


class ChannelwiseTP:
    """Alg. 2 channelwise tensor product + neighbour sum (symcon_tp_*).

        tp = ChannelwiseTP(lmax_y=3, hidden_l=(0, 1), lmax_out=3, channels=128, device=0)
        A = tp(Y, h, R, sender, receiver)     # A[N][K][(lmax_out+1)^2]; autograd gives dY, dh, dR

    Edges must be sorted by receiver. All arithmetic runs in libsymcon's kernels."""

    def __init__(self, lmax_y, hidden_l, lmax_out, channels, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("ChannelwiseTP needs a CUDA device (libsymcon has no CPU path)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.channels = channels
        with torch.cuda.device(self.device):
            self.plan = _lib.symcon_tp_build(lmax_y, list(hidden_l), lmax_out, channels, self.device.index)
        self.n_paths, self.n_y, self.n_h, self.n_out = _lib.symcon_tp_info(self.plan)
        self._ws = None

    def __del__(self):
        plan = getattr(self, "plan", None)
        if plan is not None:
            _lib.symcon_tp_destroy(plan)
            self.plan = None

    def workspace(self, N, E):
        nbytes = _lib.symcon_tp_workspace_bytes(self.plan, N, E)
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
            self._ws[:8].fill_(255)   # error word = "no error" until a call writes it
        return self._ws

    def _check(self, Y, h, R, sender, receiver):
        N, E, K = h.shape[0], sender.shape[0], self.channels
        for t in (Y, h, R):
            assert t.is_cuda and t.dtype == torch.float32 and t.is_contiguous()
        assert Y.shape == (E, self.n_y) and h.shape == (N, self.n_h, K) and R.shape == (E, self.n_paths, K)
        assert sender.dtype == torch.int32 and receiver.dtype == torch.int32 and receiver.shape == (E,)
        return N, E

    def forward_raw(self, Y, h, R, sender, receiver, A=None, prep_backward=False):
        """prep_backward=True: also build the backward's sender CSR (SYMCON_TP_PREP_BACKWARD), concurrently
        with the forward kernel, for a following backward_raw(..., reuse=True)."""
        N, E = self._check(Y, h, R, sender, receiver)
        if A is None:
            A = torch.empty((N, self.channels, self.n_out), dtype=torch.float32, device=self.device)
        ws = self.workspace(N, E)
        ptr = lambda t: t.data_ptr() if t.numel() else None
        _lib.symcon_tp_forward(self.plan, N, E, ptr(Y), ptr(h), ptr(R), ptr(sender), ptr(receiver), A.data_ptr(),
                               ws.data_ptr(), ws.numel(), _stream_ptr(self.device),
                               _lib.SYMCON_TP_PREP_BACKWARD if prep_backward else 0)
        return A

    def backward_raw(self, Y, h, R, sender, receiver, dA, need_Y=True, need_h=True, need_R=True, reuse=False):
        """reuse=True: the sender / receiver arrays are those of the last call on this workspace, unchanged
        since (SYMCON_TP_REUSE_GRAPH: the graph structure built then is kept)."""
        N, E = self._check(Y, h, R, sender, receiver)
        assert dA.dtype == torch.float32 and dA.is_contiguous() and dA.shape == (N, self.channels, self.n_out)
        dY = torch.empty_like(Y) if need_Y else None
        dh = torch.empty_like(h) if need_h else None
        dR = torch.empty_like(R) if need_R else None
        ws = self.workspace(N, E)
        ptr = lambda t: t.data_ptr() if (t is not None and t.numel()) else None
        _lib.symcon_tp_backward(self.plan, N, E, ptr(Y), ptr(h), ptr(R), ptr(sender), ptr(receiver), dA.data_ptr(),
                                ptr(dY), ptr(dh), ptr(dR), ws.data_ptr(), ws.numel(), _stream_ptr(self.device),
                                _lib.SYMCON_TP_REUSE_GRAPH if reuse else 0)
        return dY, dh, dR

    def backward2_raw(self, Y, h, R, sender, receiver, dA, uY, uh, uR):
        """(Y_bar, h_bar, R_bar, dA_bar): the TP double backward (symcon_tp_backward2), returned in the
        order of _TPBwdFn's inputs (Y, h, R, [sender, receiver,] dA)."""
        N, E = self._check(Y, h, R, sender, receiver)
        dA_bar = torch.empty((N, self.channels, self.n_out), dtype=torch.float32, device=self.device)
        Yb, hb, Rb = torch.empty_like(Y), torch.empty_like(h), torch.empty_like(R)
        nbytes = _lib.symcon_tp_workspace2_bytes(self.plan, N, E)
        ws2 = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        ws2[:8].fill_(255)
        ptr = lambda t: t.data_ptr() if (t is not None and t.numel()) else None
        _lib.symcon_tp_backward2(self.plan, N, E, ptr(Y), ptr(h), ptr(R), ptr(sender), ptr(receiver), dA.contiguous().data_ptr(),
                                 ptr(uY), ptr(uh), ptr(uR), dA_bar.data_ptr(), ptr(Yb), ptr(hb), ptr(Rb), ws2.data_ptr(),
                                 ws2.numel(), _stream_ptr(self.device))
        return Yb, hb, Rb, None, None, dA_bar

    def check_device_error(self):
        if self._ws is None:
            return 0, -1
        return _lib.symcon_tp_check_device_error(self.plan, self._ws.data_ptr(), _stream_ptr(self.device))

    def last_launch_count(self):
        return _lib.symcon_tp_last_launch_count(self.plan)

    def __call__(self, Y, h, R, sender, receiver):
        return _TPFn.apply(Y, h, R, sender, receiver, self)


class _TPFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, Y, h, R, sender, receiver, tp):
        ctx.tp = tp
        Y, h, R = Y.contiguous(), h.contiguous(), R.contiguous()
        ctx.save_for_backward(Y, h, R, sender, receiver)
        return tp.forward_raw(Y, h, R, sender, receiver)

    @staticmethod
    def backward(ctx, dA):
        Y, h, R, sender, receiver = ctx.saved_tensors
        if torch.is_grad_enabled():
            # create_graph=True (forces in the loss flow through Y and R): differentiable backward
            dY, dh, dR = _TPBwdFn.apply(Y, h, R, sender, receiver, dA.contiguous(), ctx.tp)
            return dY, dh, dR, None, None, None
        # sender / receiver are saved tensors (autograd rejects in-place changes): keep the forward's graph structure
        dY, dh, dR = ctx.tp.backward_raw(Y, h, R, sender, receiver, dA.contiguous(), *ctx.needs_input_grad[:3], reuse=True)
        return dY, dh, dR, None, None, None


class _TPBwdFn(torch.autograd.Function):
    """(Y, h, R, dA) -> (dY, dh, dR) with its own backward. The TP is linear in each of Y, h, R,
    so the second derivatives are TP passes with one input replaced by its cotangent:
      dA_bar = TP(uY, h, R) + TP(Y, uh, R) + TP(Y, h, uR)
      Y_bar  = dY|_(h := uh) + dY|_(R := uR),  h_bar = dh|_(Y := uY) + dh|_(R := uR),
      R_bar  = dR|_(Y := uY) + dR|_(h := uh)   (all with the same dA)."""

    @staticmethod
    def forward(ctx, Y, h, R, sender, receiver, dA, tp):
        ctx.tp = tp
        ctx.save_for_backward(Y, h, R, sender, receiver, dA)
        return tp.backward_raw(Y, h, R, sender, receiver, dA)

    @staticmethod
    @torch.autograd.function.once_differentiable
    def backward(ctx, uY, uh, uR):
        Y, h, R, s, r, dA = ctx.saved_tensors
        tp = ctx.tp
        z = lambda x, ref: torch.zeros_like(ref) if x is None else x.contiguous()   # absent cotangent = 0
        uY, uh, uR = z(uY, Y), z(uh, h), z(uR, R)
        # all six passes and their sums run in libsymcon (symcon_tp_backward2)
        return tp.backward2_raw(Y, h, R, s, r, dA, uY, uh, uR) + (None,)
