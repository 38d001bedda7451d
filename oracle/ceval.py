"""ctypes wrapper for oracle/csrc/oracle_eval.c (oracle; test infrastructure only).

The C loop evaluates the same raw ordered-tuple terms as oracle/contraction.py
(which builds them); tests/test_oracle_ceval.py pins the two against each other.
"""
import ctypes
import os
import subprocess

import numpy as np

from .contraction import Problem

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "oracle_eval.c")
_LIB = os.path.join(_HERE, "csrc", "liboracle_eval.so")


def build():
    if not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC])
    return _LIB


class _Tables(ctypes.Structure):
    _fields_ = [("n_terms", ctypes.c_int64), ("n_lm", ctypes.c_int64), ("out_per_ch", ctypes.c_int64),
                ("n_paths", ctypes.c_int64)] + [(n, ctypes.c_void_p) for n in
                                                ("col", "nu", "tup", "blk", "wid", "mpos", "u")]


class OracleC:
    def __init__(self, prob: Problem):
        self.lib = ctypes.CDLL(build())
        self.prob = prob
        rows = []
        blk = {}
        off = 0
        for L in prob.out_L:
            blk[L] = off
            off += 2 * L + 1
        for p in prob.paths:
            for M, ts, u in p.terms:
                tp = list(ts) + [0] * (4 - len(ts))   # up to nu = 4 (correlation 4, reading s4b)
                rows.append((p.col, p.nu, tp, blk[p.L], 2 * p.L + 1, M + p.L, u))
        self._arr = {
            "col": np.array([r[0] for r in rows], np.int32),
            "nu": np.array([r[1] for r in rows], np.int32),
            "tup": np.array([r[2] for r in rows], np.int32).reshape(-1),
            "blk": np.array([r[3] for r in rows], np.int32),
            "wid": np.array([r[4] for r in rows], np.int32),
            "mpos": np.array([r[5] for r in rows], np.int32),
            "u": np.array([r[6] for r in rows], np.float64),
        }
        self.t = _Tables(len(rows), prob.n_lm, prob.out_per_channel, prob.n_paths,
                         *[self._arr[n].ctypes.data for n in ("col", "nu", "tup", "blk", "wid", "mpos", "u")])
        self.n_terms = len(rows)
        self.lib.oracle_num_threads.restype = ctypes.c_int
        # use every core of this process's affinity mask (torchrun exports OMP_NUM_THREADS=1)
        self.lib.oracle_set_threads(ctypes.c_int(len(os.sched_getaffinity(0))))

    def threads(self):
        return self.lib.oracle_num_threads()

    @staticmethod
    def _f32(x):
        return np.ascontiguousarray(x, dtype=np.float32)

    def forward(self, A, W, node_elem):
        A, W = self._f32(A), self._f32(W)
        ne = np.ascontiguousarray(node_elem, dtype=np.int32)
        N, K, _ = A.shape
        B = np.zeros((N, self.prob.out_dim(K)))
        self.lib.oracle_forward(ctypes.byref(self.t), ctypes.c_int64(N), ctypes.c_int64(K),
                                A.ctypes.data_as(ctypes.c_void_p), W.ctypes.data_as(ctypes.c_void_p),
                                ne.ctypes.data_as(ctypes.c_void_p), B.ctypes.data_as(ctypes.c_void_p))
        return B

    def backward(self, A, W, node_elem, dB, want_dA=True, want_dW=True):
        A, W, dB = self._f32(A), self._f32(W), self._f32(dB)
        ne = np.ascontiguousarray(node_elem, dtype=np.int32)
        N, K, _ = A.shape
        E = W.shape[0]
        dA = np.zeros(A.shape) if want_dA else None
        dW = np.zeros(W.shape) if want_dW else None
        p = lambda x: x.ctypes.data_as(ctypes.c_void_p) if x is not None else None
        self.lib.oracle_backward(ctypes.byref(self.t), ctypes.c_int64(N), ctypes.c_int64(K), ctypes.c_int64(E),
                                 p(A), p(W), p(ne), p(dB), p(dA), p(dW))
        return dA, dW

    def backward2(self, A, W, node_elem, dB, uA, want_dB=True, want_A=True, want_W=True):
        A, W, dB, uA = self._f32(A), self._f32(W), self._f32(dB), self._f32(uA)
        ne = np.ascontiguousarray(node_elem, dtype=np.int32)
        N, K, _ = A.shape
        E = W.shape[0]
        dBb = np.zeros((N, self.prob.out_dim(K))) if want_dB else None
        Ab = np.zeros(A.shape) if want_A else None
        Wb = np.zeros(W.shape) if want_W else None
        p = lambda x: x.ctypes.data_as(ctypes.c_void_p) if x is not None else None
        self.lib.oracle_backward2(ctypes.byref(self.t), ctypes.c_int64(N), ctypes.c_int64(K), ctypes.c_int64(E),
                                  p(A), p(W), p(ne), p(dB), p(uA), p(dBb), p(Ab), p(Wb))
        return dBb, Ab, Wb
