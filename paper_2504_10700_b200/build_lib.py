"""Build libsymcon.so in-tree (nvcc for sm_100a + g++), and optionally precompile the
generated kernels of the preset configurations into the in-tree cubin cache.

    python -m paper_2504_10700_b200.build_lib [--precompile]
"""
import ctypes
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libsymcon.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES = ["cg.cpp", "builder.cpp", "codegen.cpp", "codegen_simple.cpp", "pack.cpp", "api.cpp", "tp.cpp", "bucket.cu", "tp_static.cu", "peer.cu"]

# (lmax_in, correlation, out_L): BASELINE configs + the corr-1/2 cases the tests use
PRESETS = [(3, 3, (0,)), (3, 3, (0, 1)), (3, 3, (0, 1, 2)), (3, 1, (0, 1, 2, 3)), (3, 2, (0,)),
           (3, 2, (0, 1)), (2, 3, (0, 1)), (1, 3, (0, 1)), (3, 3, (1,)), (0, 3, (0,)), (3, 2, (2, 3)),
           (2, 3, (0, 1, 2, 3))]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose=False):
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, "internal.h"), os.path.join(CSRC, "kernels.h"),
                                                      os.path.join(ROOT, "include", "symcon.h"), __file__]
    if not _newer(OUT, deps):
        return OUT
    objdir = os.path.join(HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(objdir, s + ".o")
        if s.endswith(".cu"):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-Xptxas", "-v", "-std=c++17", "-Xcompiler", "-fPIC", "-c", src, "-o", obj]
        else:
            cmd = [NVCC, "-O3", "-std=c++17", "-Xcompiler", "-fPIC,-Wall", "-I" + os.path.join(CUDA, "include"),
                   "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr)
        objs.append(obj)
    link = [NVCC, *ARCH, "-shared", "-o", OUT, *objs, "-L" + os.path.join(CUDA, "lib64"),
            "-lnvrtc_static", "-lnvrtc-builtins_static", "-lnvptxcompiler_static", "-lcudart_static", "-ldl", "-lrt",
            "-lpthread", "-Xlinker", "--exclude-libs,ALL"]
    r = subprocess.run(link, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
    return OUT


# channelwise TP (lmax_y, hidden_l, lmax_out, K): the bench shape and the test configurations
TP_PRESETS = [(3, (0, 1), 3, 128), (3, (0, 1), 3, 64), (3, (0, 1), 3, 32), (3, (0, 1), 3, 6), (3, (0,), 3, 64),
              (3, (0, 1, 2), 3, 32), (2, (0, 1), 2, 13), (2, (0, 1), 2, 96), (1, (1,), 1, 40), (3, (0, 1, 2, 3), 3, 33),
              (2, (0,), 2, 1), (0, (0, 1, 2), 2, 16)]


def precompile_tp(presets=TP_PRESETS):
    lib = ctypes.CDLL(build())
    lib.symcon_tp_precompile.restype = ctypes.c_int
    lib.symcon_last_error.restype = ctypes.c_char_p
    for ly, hid, lo, k in presets:
        arr = (ctypes.c_int * len(hid))(*hid)
        if lib.symcon_tp_precompile(ly, arr, len(hid), lo, k) != 0:
            raise RuntimeError(f"tp precompile {ly},{hid},{lo},{k} failed: {lib.symcon_last_error().decode()}")


# fp64 plans (SYMCON_F64) compiled at build time: the BASELINE shapes and the fp64 test configurations
PRESETS_F64 = [(3, 3, (0,)), (3, 3, (0, 1)), (3, 3, (0, 1, 2)), (2, 2, (0, 1)),
               (3, 4, (0,)), (2, 4, (0, 1))]
# correlation 4 (plain scalar kernels, codegen_simple.cpp; NVRTC ~100 s for (3, 4, (0, 1)))
PRESETS_C4 = [(3, 4, (0,)), (3, 4, (0, 1)), (2, 4, (0, 1, 2))]


def precompile(presets=PRESETS + PRESETS_C4, presets_f64=PRESETS_F64):
    lib = ctypes.CDLL(build())
    lib.symcon_precompile_ex.restype = ctypes.c_int
    lib.symcon_precompile_ex.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int32,
                                         ctypes.c_char_p, ctypes.c_size_t]
    lib.symcon_last_error.restype = ctypes.c_char_p
    paths = []
    for dtype, plist in ((0, presets), (1, presets_f64)):
        for lmax, corr, outs in plist:
            arr = (ctypes.c_int * len(outs))(*outs)
            buf = ctypes.create_string_buffer(4096)
            s = lib.symcon_precompile_ex(lmax, corr, arr, len(outs), dtype, buf, 4096)
            if s != 0:
                raise RuntimeError(f"precompile {lmax},{corr},{outs} dtype {dtype} failed: {lib.symcon_last_error().decode()}")
            paths.append(buf.value.decode())
    return paths


if __name__ == "__main__":
    print(build(verbose=True))
    if "--precompile" in sys.argv:
        for p in precompile():
            print(p)
