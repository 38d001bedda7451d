"""Thin ctypes binding of libsymcon.so (include/symcon.h). Argument marshalling only.

Names follow the C ABI. Device pointers are passed as integers (e.g. tensor.data_ptr()),
streams as cudaStream_t integers (torch.cuda.current_stream().cuda_stream). Every step of
the contraction runs in the library's CUDA kernels; there is no CPU fallback: if the
library is missing this module raises at import time.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsymcon.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"libsymcon.so not built at {LIB_PATH}: run `python -m paper_2504_10700_b200.build_lib` "
                      "(or __graft_entry__.build())")

lib = ctypes.CDLL(LIB_PATH)

SYMCON_OK, SYMCON_EINVAL, SYMCON_EUNSUPPORTED, SYMCON_ECUDA, SYMCON_ENOMEM, SYMCON_EELEMENT, SYMCON_ETIMEOUT = range(7)

EXPORTS = ["symcon_build_tables", "symcon_plan_info", "symcon_plan_path", "symcon_plan_sym_table", "symcon_plan_sym_table4", "symcon_real_cg",
           "symcon_workspace_bytes", "symcon_forward", "symcon_backward", "symcon_backward_ex", "symcon_backward2", "symcon_check_device_error",
           "symcon_last_launch_count", "symcon_destroy", "symcon_status_string", "symcon_last_error",
           "symcon_pack_balanced", "symcon_precompile", "symcon_plan_source", "symcon_profile_enable",
           "symcon_profile_reset", "symcon_profile_read", "symcon_tp_build", "symcon_tp_info", "symcon_tp_path",
           "symcon_tp_workspace_bytes", "symcon_tp_forward", "symcon_tp_backward", "symcon_tp_check_device_error",
           "symcon_tp_last_launch_count", "symcon_tp_source", "symcon_tp_destroy", "symcon_peer_allreduce",
           "symcon_tp_precompile", "symcon_peer_allreduce_dev", "symcon_peer_allreduce_ex", "symcon_peer_check",
           "symcon_peer_allreduce_emulate", "symcon_backward2_ex", "symcon_tp_backward2", "symcon_tp_workspace2_bytes",
           "symcon_tp_forward_ex", "symcon_tp_backward_ex", "symcon_tp_backward2_ex", "symcon_plan_sym_table4",
           "symcon_build_tables_ex", "symcon_forward_f64", "symcon_backward_f64", "symcon_precompile_ex"]
SYMCON_F32, SYMCON_F64 = 0, 1


class SymconInfo(ctypes.Structure):
    _fields_ = [("lmax_in", ctypes.c_int32), ("correlation", ctypes.c_int32), ("n_out", ctypes.c_int32),
                ("num_elements", ctypes.c_int32), ("channels", ctypes.c_int32), ("out_L", ctypes.c_int32 * 4),
                ("eta", (ctypes.c_int32 * 4) * 4), ("n_paths", ctypes.c_int64), ("weight_numel", ctypes.c_int64),
                ("in_dim", ctypes.c_int64), ("out_dim", ctypes.c_int64), ("n_raw_terms", ctypes.c_int64),
                ("n_sym_terms", ctypes.c_int64), ("n_fold", ctypes.c_int64), ("n_monomials", ctypes.c_int64),
                ("device", ctypes.c_int32), ("reserved", ctypes.c_int32)]


_vp, _i64, _i32, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_size_t
lib.symcon_build_tables.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_int, ctypes.POINTER(_vp)]
lib.symcon_plan_info.argtypes = [_vp, ctypes.POINTER(SymconInfo)]
lib.symcon_plan_path.argtypes = [_vp, _i64] + [ctypes.POINTER(_i32)] * 5
lib.symcon_plan_sym_table.argtypes = [_vp, ctypes.POINTER(_i64), _vp, _vp, _vp, _vp, _vp]
lib.symcon_plan_sym_table4.argtypes = [_vp, ctypes.POINTER(_i64), _vp, _vp, _vp, _vp, _vp]
lib.symcon_real_cg.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]
lib.symcon_workspace_bytes.argtypes = [_vp, _i64]
lib.symcon_workspace_bytes.restype = _sz
lib.symcon_forward.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
lib.symcon_backward.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
lib.symcon_backward_ex.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.c_uint32, _vp]
lib.symcon_backward2.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.c_uint32, _vp]
lib.symcon_backward2_ex.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.c_uint32, _vp]
lib.symcon_backward2_ex.restype = ctypes.c_int
SYMCON_REUSE_BUCKETS, SYMCON_REUSE_FOLD = 1, 2
lib.symcon_check_device_error.argtypes = [_vp, _vp, _vp, ctypes.POINTER(_i64)]
lib.symcon_last_launch_count.argtypes = [_vp]
lib.symcon_last_launch_count.restype = _i32
lib.symcon_destroy.argtypes = [_vp]
lib.symcon_destroy.restype = None
lib.symcon_status_string.argtypes = [ctypes.c_int]
lib.symcon_status_string.restype = ctypes.c_char_p
lib.symcon_last_error.restype = ctypes.c_char_p
lib.symcon_pack_balanced.argtypes = [_vp, _i64, _i64, _i32, _vp, _vp, _i64, ctypes.POINTER(_i64)]
lib.symcon_precompile.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                  ctypes.c_char_p, _sz]
lib.symcon_plan_source.argtypes = [_vp, ctypes.c_char_p, _sz]
lib.symcon_plan_source.restype = _sz
lib.symcon_profile_enable.argtypes = [_vp, ctypes.c_int]
lib.symcon_profile_reset.argtypes = [_vp]
lib.symcon_profile_read.argtypes = [_vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(_i64),
                                    ctypes.POINTER(ctypes.c_double)]
lib.symcon_profile_read.restype = _i32
for _n in ("symcon_profile_enable", "symcon_profile_reset", "symcon_build_tables", "symcon_plan_info", "symcon_plan_path", "symcon_plan_sym_table", "symcon_plan_sym_table4",
           "symcon_real_cg", "symcon_forward", "symcon_backward", "symcon_backward_ex", "symcon_backward2", "symcon_check_device_error", "symcon_pack_balanced",
           "symcon_precompile"):
    getattr(lib, _n).restype = ctypes.c_int


PROFILE_MAX = 12  # SYMCON_PROFILE_MAX


class SymconError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = lib.symcon_last_error().decode(errors="replace")
        super().__init__(f"{where}: {lib.symcon_status_string(status).decode()} ({msg})")


def check(status, where):
    if status != SYMCON_OK:
        raise SymconError(status, where)


def symcon_build_tables(lmax_in, correlation, out_L, num_elements, channels, device):
    arr = (ctypes.c_int * len(out_L))(*out_L)
    plan = _vp()
    check(lib.symcon_build_tables(lmax_in, correlation, arr, len(out_L), num_elements, channels, device,
                                  ctypes.byref(plan)), "symcon_build_tables")
    return plan


lib.symcon_build_tables_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_int, _i32, ctypes.POINTER(_vp)]
lib.symcon_build_tables_ex.restype = ctypes.c_int
lib.symcon_forward_f64.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
lib.symcon_forward_f64.restype = ctypes.c_int
lib.symcon_backward_f64.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.c_uint32, _vp]
lib.symcon_backward_f64.restype = ctypes.c_int
lib.symcon_precompile_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, _i32,
                                     ctypes.c_char_p, _sz]
lib.symcon_precompile_ex.restype = ctypes.c_int


def symcon_build_tables_ex(lmax_in, correlation, out_L, num_elements, channels, device, dtype):
    arr = (ctypes.c_int * len(out_L))(*out_L)
    plan = _vp()
    check(lib.symcon_build_tables_ex(lmax_in, correlation, arr, len(out_L), num_elements, channels, device, dtype,
                                     ctypes.byref(plan)), "symcon_build_tables_ex")
    return plan


def symcon_forward_f64(plan, num_nodes, A, W, node_elem, B, ws, ws_bytes, stream):
    check(lib.symcon_forward_f64(plan, num_nodes, A, W, node_elem, B, ws, ws_bytes, stream), "symcon_forward_f64")


def symcon_backward_f64(plan, num_nodes, A, W, node_elem, dB, dA, dW, ws, ws_bytes, flags, stream):
    check(lib.symcon_backward_f64(plan, num_nodes, A, W, node_elem, dB, dA, dW, ws, ws_bytes, flags, stream),
          "symcon_backward_f64")


def symcon_precompile_ex(lmax_in, correlation, out_L, dtype):
    arr = (ctypes.c_int * len(out_L))(*out_L)
    buf = ctypes.create_string_buffer(4096)
    check(lib.symcon_precompile_ex(lmax_in, correlation, arr, len(out_L), dtype, buf, 4096), "symcon_precompile_ex")
    return buf.value.decode()


def symcon_plan_info(plan):
    info = SymconInfo()
    check(lib.symcon_plan_info(plan, ctypes.byref(info)), "symcon_plan_info")
    return info


def symcon_plan_path(plan, col):
    L, nu, eta = _i32(), _i32(), _i32()
    ls, mids = (_i32 * 4)(), (_i32 * 3)()
    check(lib.symcon_plan_path(plan, col, ctypes.byref(L), ctypes.byref(nu), ctypes.byref(eta), ls, mids),
          "symcon_plan_path")
    return L.value, nu.value, eta.value, tuple(ls[:nu.value]), tuple(mids[:max(nu.value - 1, 0)])


def symcon_plan_sym_table(plan, width=3):
    """(L, M, mono[n, width], col, value); width 4 calls symcon_plan_sym_table4 (correlation 4)."""
    import numpy as np
    fn = lib.symcon_plan_sym_table if width == 3 else lib.symcon_plan_sym_table4
    n = _i64(0)
    check(fn(plan, ctypes.byref(n), None, None, None, None, None), "symcon_plan_sym_table")
    L = np.zeros(n.value, np.int32)
    M = np.zeros(n.value, np.int32)
    mono = np.zeros((n.value, width), np.int32)
    col = np.zeros(n.value, np.int32)
    val = np.zeros(n.value, np.float64)
    check(fn(plan, ctypes.byref(n), L.ctypes.data, M.ctypes.data, mono.ctypes.data, col.ctypes.data, val.ctypes.data),
          "symcon_plan_sym_table")
    return L, M, mono, col, val


def symcon_real_cg(l1, l2, L):
    import numpy as np
    out = np.zeros((2 * L + 1, 2 * l1 + 1, 2 * l2 + 1), np.float64)
    check(lib.symcon_real_cg(l1, l2, L, out.ctypes.data), "symcon_real_cg")
    return out


def symcon_plan_source(plan):
    n = lib.symcon_plan_source(plan, None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib.symcon_plan_source(plan, buf, n + 1)
    return buf.value.decode()


def symcon_workspace_bytes(plan, num_nodes):
    return lib.symcon_workspace_bytes(plan, num_nodes)


def symcon_forward(plan, num_nodes, A, W, node_elem, B, ws, ws_bytes, stream):
    check(lib.symcon_forward(plan, num_nodes, A, W, node_elem, B, ws, ws_bytes, stream), "symcon_forward")


def symcon_backward(plan, num_nodes, A, W, node_elem, dB, dA, dW, ws, ws_bytes, stream):
    check(lib.symcon_backward(plan, num_nodes, A, W, node_elem, dB, dA, dW, ws, ws_bytes, stream), "symcon_backward")


def symcon_backward_ex(plan, num_nodes, A, W, node_elem, dB, dA, dW, ws, ws_bytes, flags, stream):
    check(lib.symcon_backward_ex(plan, num_nodes, A, W, node_elem, dB, dA, dW, ws, ws_bytes, flags, stream),
          "symcon_backward_ex")


def symcon_backward2(plan, num_nodes, A, W, node_elem, dB, uA, dB_bar, A_bar, W_bar, ws, ws_bytes, flags, stream):
    check(lib.symcon_backward2(plan, num_nodes, A, W, node_elem, dB, uA, dB_bar, A_bar, W_bar, ws, ws_bytes, flags, stream),
          "symcon_backward2")


def symcon_backward2_ex(plan, num_nodes, A, W, node_elem, dB, uA, uW, dB_bar, A_bar, W_bar, ws, ws_bytes, flags, stream):
    check(lib.symcon_backward2_ex(plan, num_nodes, A, W, node_elem, dB, uA, uW, dB_bar, A_bar, W_bar, ws, ws_bytes, flags,
                                  stream), "symcon_backward2_ex")


def symcon_check_device_error(plan, ws, stream):
    bad = _i64(-1)
    s = lib.symcon_check_device_error(plan, ws, stream, ctypes.byref(bad))
    return s, bad.value


def symcon_last_launch_count(plan):
    return lib.symcon_last_launch_count(plan)


def symcon_destroy(plan):
    lib.symcon_destroy(plan)


def symcon_pack_balanced(sizes, capacity, workers):
    """Alg. 1 on host (C++). Returns (bin_offsets, graph_ids) as numpy int64 arrays."""
    import numpy as np
    sizes = np.ascontiguousarray(sizes, dtype=np.int64)
    n = len(sizes)
    nb = _i64(0)
    s = lib.symcon_pack_balanced(sizes.ctypes.data, n, capacity, workers, None, None, 0, ctypes.byref(nb))
    if s not in (SYMCON_OK, SYMCON_ENOMEM):
        check(s, "symcon_pack_balanced")
    offs = np.zeros(nb.value + 1, np.int64)
    ids = np.zeros(max(n, 1), np.int64)
    check(lib.symcon_pack_balanced(sizes.ctypes.data, n, capacity, workers, offs.ctypes.data, ids.ctypes.data,
                                   nb.value, ctypes.byref(nb)), "symcon_pack_balanced")
    return offs, ids[:n]


def symcon_precompile(lmax_in, correlation, out_L):
    arr = (ctypes.c_int * len(out_L))(*out_L)
    buf = ctypes.create_string_buffer(4096)
    check(lib.symcon_precompile(lmax_in, correlation, arr, len(out_L), buf, 4096), "symcon_precompile")
    return buf.value.decode()


def symcon_profile_enable(plan, on=1):
    check(lib.symcon_profile_enable(plan, int(on)), "symcon_profile_enable")


def symcon_profile_reset(plan):
    check(lib.symcon_profile_reset(plan), "symcon_profile_reset")


def symcon_profile_read(plan):
    """{kernel name: (launches, total ms)} of the launch timer (synchronises)."""
    names = (ctypes.c_char_p * PROFILE_MAX)()
    counts = (_i64 * PROFILE_MAX)()
    ms = (ctypes.c_double * PROFILE_MAX)()
    n = lib.symcon_profile_read(plan, names, counts, ms)
    return {names[i].decode(): (int(counts[i]), float(ms[i])) for i in range(n)}


# ------------------------------------------------------------ channelwise TP (symcon_tp_*)
lib.symcon_tp_build.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.POINTER(_vp)]
lib.symcon_tp_info.argtypes = [_vp] + [ctypes.POINTER(_i32)] * 4
lib.symcon_tp_path.argtypes = [_vp, _i32] + [ctypes.POINTER(_i32)] * 3
lib.symcon_tp_workspace_bytes.argtypes = [_vp, _i64, _i64]
lib.symcon_tp_workspace_bytes.restype = _sz
lib.symcon_tp_forward.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
lib.symcon_tp_backward.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, _vp]
lib.symcon_tp_check_device_error.argtypes = [_vp, _vp, _vp, ctypes.POINTER(_i64)]
lib.symcon_tp_last_launch_count.argtypes = [_vp]
lib.symcon_tp_last_launch_count.restype = _i32
lib.symcon_tp_source.argtypes = [_vp, ctypes.c_char_p, _sz]
lib.symcon_tp_source.restype = _sz
lib.symcon_tp_destroy.argtypes = [_vp]
lib.symcon_tp_destroy.restype = None
for _n in ("symcon_tp_build", "symcon_tp_info", "symcon_tp_path", "symcon_tp_forward", "symcon_tp_backward",
           "symcon_tp_check_device_error"):
    getattr(lib, _n).restype = ctypes.c_int


def symcon_tp_build(lmax_y, hidden_l, lmax_out, channels, device):
    arr = (ctypes.c_int * len(hidden_l))(*hidden_l)
    plan = _vp()
    check(lib.symcon_tp_build(lmax_y, arr, len(hidden_l), lmax_out, channels, device, ctypes.byref(plan)),
          "symcon_tp_build")
    return plan


def symcon_tp_info(plan):
    v = [_i32() for _ in range(4)]
    check(lib.symcon_tp_info(plan, *[ctypes.byref(x) for x in v]), "symcon_tp_info")
    return tuple(x.value for x in v)   # n_paths, n_y, n_h, n_out


def symcon_tp_path(plan, p):
    v = [_i32() for _ in range(3)]
    check(lib.symcon_tp_path(plan, p, *[ctypes.byref(x) for x in v]), "symcon_tp_path")
    return tuple(x.value for x in v)


def symcon_tp_workspace_bytes(plan, num_nodes, num_edges):
    return lib.symcon_tp_workspace_bytes(plan, num_nodes, num_edges)


lib.symcon_tp_workspace2_bytes.argtypes = [_vp, _i64, _i64]
lib.symcon_tp_workspace2_bytes.restype = _sz
lib.symcon_tp_backward2.argtypes = [_vp, _i64, _i64] + [_vp] * 14 + [_sz, _vp]
lib.symcon_tp_backward2.restype = ctypes.c_int


def symcon_tp_workspace2_bytes(plan, num_nodes, num_edges):
    return lib.symcon_tp_workspace2_bytes(plan, num_nodes, num_edges)


def symcon_tp_backward2(plan, N, E, Y, h, R, sender, receiver, dA, uY, uh, uR, dA_bar, Y_bar, h_bar, R_bar, ws, ws_bytes,
                        stream, flags=0):
    check(lib.symcon_tp_backward2_ex(plan, N, E, Y, h, R, sender, receiver, dA, uY, uh, uR, dA_bar, Y_bar, h_bar, R_bar, ws,
                                     ws_bytes, flags, stream), "symcon_tp_backward2")


SYMCON_TP_REUSE_GRAPH = 4
SYMCON_TP_PREP_BACKWARD = 8
lib.symcon_tp_forward_ex.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz, ctypes.c_uint32, _vp]
lib.symcon_tp_forward_ex.restype = ctypes.c_int
lib.symcon_tp_backward_ex.argtypes = [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _sz,
                                      ctypes.c_uint32, _vp]
lib.symcon_tp_backward_ex.restype = ctypes.c_int
lib.symcon_tp_backward2_ex.argtypes = [_vp, _i64, _i64] + [_vp] * 14 + [_sz, ctypes.c_uint32, _vp]
lib.symcon_tp_backward2_ex.restype = ctypes.c_int


def symcon_tp_forward(plan, N, E, Y, h, R, sender, receiver, A, ws, ws_bytes, stream, flags=0):
    check(lib.symcon_tp_forward_ex(plan, N, E, Y, h, R, sender, receiver, A, ws, ws_bytes, flags, stream),
          "symcon_tp_forward")


def symcon_tp_backward(plan, N, E, Y, h, R, sender, receiver, dA, dY, dh, dR, ws, ws_bytes, stream, flags=0):
    check(lib.symcon_tp_backward_ex(plan, N, E, Y, h, R, sender, receiver, dA, dY, dh, dR, ws, ws_bytes, flags, stream),
          "symcon_tp_backward")


def symcon_tp_check_device_error(plan, ws, stream):
    bad = _i64(-1)
    s = lib.symcon_tp_check_device_error(plan, ws, stream, ctypes.byref(bad))
    return s, bad.value


def symcon_tp_source(plan):
    n = lib.symcon_tp_source(plan, None, 0)
    buf = ctypes.create_string_buffer(n + 1)
    lib.symcon_tp_source(plan, buf, n + 1)
    return buf.value.decode()


def symcon_tp_destroy(plan):
    lib.symcon_tp_destroy(plan)


def symcon_tp_last_launch_count(plan):
    return lib.symcon_tp_last_launch_count(plan)


# ------------------------------------------------------------ dW all-reduce over peer memory
lib.symcon_peer_allreduce.argtypes = [_vp, _vp, _i32, _i32, _i64, ctypes.c_uint32, _vp, _vp, _vp]
lib.symcon_peer_allreduce.restype = ctypes.c_int


def symcon_peer_allreduce(bufs, pads, rank, n, epoch, out, err, stream):
    world = len(bufs)
    b = (_vp * world)(*bufs)
    p = (_vp * world)(*pads)
    check(lib.symcon_peer_allreduce(b, p, world, rank, n, epoch, out, err, stream), "symcon_peer_allreduce")


lib.symcon_peer_allreduce_dev.argtypes = [_vp, _vp, _i32, _i32, _i64, _vp, _vp, _vp, _vp]
lib.symcon_peer_allreduce_dev.restype = ctypes.c_int


def symcon_peer_allreduce_dev(bufs, pads, rank, n, epoch_counter, out, err, stream):
    world = len(bufs)
    b = (_vp * world)(*bufs)
    p = (_vp * world)(*pads)
    check(lib.symcon_peer_allreduce_dev(b, p, world, rank, n, epoch_counter, out, err, stream),
          "symcon_peer_allreduce_dev")


lib.symcon_peer_allreduce_ex.argtypes = [_vp, _vp, _i32, _i32, _i64, ctypes.c_uint32, _vp, _i32, _i64, _vp, _vp, _vp]
lib.symcon_peer_allreduce_ex.restype = ctypes.c_int


def symcon_peer_allreduce_ex(bufs, pads, rank, n, epoch, epoch_counter, algo, spin_limit, out, err, stream):
    world = len(bufs)
    b = (_vp * world)(*bufs)
    p = (_vp * world)(*pads)
    check(lib.symcon_peer_allreduce_ex(b, p, world, rank, n, epoch, epoch_counter, algo, spin_limit, out, err, stream),
          "symcon_peer_allreduce_ex")


lib.symcon_peer_check.argtypes = [_vp, _vp]
lib.symcon_peer_check.restype = ctypes.c_int


def symcon_peer_check(err, stream):
    """Synchronises; raises SymconError(SYMCON_ETIMEOUT) if an all-reduce barrier timed out."""
    check(lib.symcon_peer_check(err, stream), "symcon_peer_check")


lib.symcon_peer_allreduce_emulate.argtypes = [_vp, _vp, _vp, _i32, _i64, ctypes.c_uint32, _i32, _i64, _vp, _vp]
lib.symcon_peer_allreduce_emulate.restype = ctypes.c_int


def symcon_peer_allreduce_emulate(bufs, pads, outs, n, epoch, algo, spin_limit, err, stream):
    world = len(bufs)
    b, p, o = (_vp * world)(*bufs), (_vp * world)(*pads), (_vp * world)(*outs)
    check(lib.symcon_peer_allreduce_emulate(b, p, o, world, n, epoch, algo, spin_limit, err, stream),
          "symcon_peer_allreduce_emulate")
