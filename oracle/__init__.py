"""CPU oracle for the online-ABFT GEMM of arXiv 2305.01024 — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  It shares no
code with the CUDA path (``paper_2305_01024_b200``) and never imports it.

The arithmetic lives in ``ftgemm_oracle.c`` (plain C, FP64); this module only
marshals numpy arrays into it.  See that file's header for the passage each step
follows.  Parity pins live in ``tests/test_oracle.py``.

Pinned functions: ``ftgemm`` (product, encode, references, verify, locate,
correct, output rounding), ``encode_col``, ``encode_row``, ``gemm_f64``,
``double_to_bf16``.  None is "parity unpinned" (see DESIGN.md §Oracle pins).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ftgemm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ACC_FP64, ACC_FP32SEQ = 0, 1
OUT_F32, OUT_BF16 = 0, 1
FT_OFF, FT_DETECT, FT_CORRECT, FT_DETECT_ROWS = 0, 1, 2, 3
INJ_FLIP, INJ_ADD = 0, 1
TGT_ACC, TGT_ROW_REF, TGT_COL_REF = 0, 1, 2
EV_CORRECTED, EV_CHECKSUM_ONLY, EV_UNCORRECTABLE, EV_LOCATED, EV_DETECTED = 1, 2, 3, 4, 5


class Inject(C.Structure):
    _fields_ = [("row", C.c_int64), ("col", C.c_int64), ("k_elem", C.c_int64),
                ("bit", C.c_int32), ("mode", C.c_int32), ("target", C.c_int32),
                ("addend", C.c_float)]


class Event(C.Structure):
    _fields_ = [("row", C.c_int64), ("col", C.c_int64),
                ("tile_m", C.c_int32), ("tile_n", C.c_int32), ("kind", C.c_int32),
                ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("k_checked", C.c_int32),
                ("resid_row", C.c_double), ("resid_col", C.c_double),
                ("tau_row", C.c_double), ("tau_col", C.c_double)]


class Counts(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("tiles_checked", "tiles_detected", "corrected",
                                         "checksum_only", "uncorrectable", "located",
                                         "events", "dropped")]


class Problem(C.Structure):
    _fields_ = [("M", C.c_int64), ("N", C.c_int64), ("K", C.c_int64),
                ("alpha", C.c_double), ("beta", C.c_double),
                ("A", C.c_void_p), ("lda", C.c_int64),
                ("B", C.c_void_p), ("ldb", C.c_int64),
                ("Cin", C.c_void_p), ("ldc", C.c_int64),
                ("out_dtype", C.c_int32), ("acc_mode", C.c_int32),
                ("Cout", C.c_void_p),
                ("tile_m", C.c_int64), ("tile_n", C.c_int64), ("bk", C.c_int64),
                ("u_acc", C.c_double), ("lambda1", C.c_double), ("lambda2", C.c_double),
                ("ft_level", C.c_int32), ("n_inj", C.c_int32),
                ("inj", C.c_void_p),
                ("counts", C.c_void_p),
                ("events", C.c_void_p), ("max_events", C.c_int32), ("pad0", C.c_int32),
                ("P_out", C.c_void_p), ("resid_row", C.c_void_p), ("resid_col", C.c_void_p),
                ("tau_row", C.c_void_p), ("tau_col", C.c_void_p), ("ks", C.c_int64)]


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, OpenMP).  -ffp-contract=off keeps every FP64
    expression exactly as written; fmaf() is the only fused operation."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC",
               "-std=c11", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.oracle_ftgemm.argtypes = [C.POINTER(Problem)]
        _lib.oracle_ftgemm.restype = C.c_int
        _lib.oracle_encode_col.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        _lib.oracle_encode_row.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p]
        _lib.oracle_gemm_f64.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_double, C.c_void_p, C.c_int64,
                                         C.c_void_p, C.c_int64, C.c_double, C.c_void_p, C.c_int64, C.c_void_p]
        _lib.oracle_double_to_bf16.argtypes = [C.c_double]
        _lib.oracle_double_to_bf16.restype = C.c_uint16
        _lib.oracle_num_threads.restype = C.c_int
    return _lib


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


@dataclass
class Result:
    C: np.ndarray            # output (float32 values; BF16 outputs given as uint16 bits in C_bits)
    C_bits: np.ndarray | None
    P: np.ndarray            # FP64 accumulator after injection / correction
    counts: dict
    events: list
    resid_row: np.ndarray    # M x tiles_n
    resid_col: np.ndarray    # tiles_m x N
    tau_row: np.ndarray
    tau_col: np.ndarray


def ftgemm(A, B, Cin=None, *, alpha=1.0, beta=0.0, out="f32", acc="fp64",
           tile_m=128, tile_n=128, bk=8, u_acc=2.0 ** -24, lambda1=16.0, lambda2=32.0,
           ft_level=FT_CORRECT, injections=(), max_events=4096, ks=0) -> Result:
    """Run the oracle on float32 operand values A (MxK), B (KxN), C_in (MxN).

    injections: iterable of dicts/tuples (row, col, k_elem, bit, mode, target, addend).
    ks > 0: online verification after every ks of K (FP64 mode).
    """
    assert ks == 0 or acc == "fp64"
    A = _f32(A); B = _f32(B)
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    Cin_a = _f32(Cin) if Cin is not None else None
    if beta != 0.0:
        assert Cin_a is not None and Cin_a.shape == (M, N)
    if out == "f32":
        Cout = np.zeros((M, N), dtype=np.float32)
    else:
        Cout = np.zeros((M, N), dtype=np.uint16)
    tm = -(-M // tile_m)
    tn = -(-N // tile_n)
    P = np.zeros((M, N), dtype=np.float64)
    rr = np.full((M, tn), np.nan); tr = np.full((M, tn), np.nan)
    rc = np.full((tm, N), np.nan); tc = np.full((tm, N), np.nan)
    inj = list(injections)
    inj_arr = (Inject * max(1, len(inj)))()
    for i, x in enumerate(inj):
        if isinstance(x, dict):
            x = (x["row"], x["col"], x["k_elem"], x.get("bit", 0), x.get("mode", INJ_FLIP),
                 x.get("target", TGT_ACC), x.get("addend", 0.0))
        inj_arr[i] = Inject(*x)
    counts = Counts()
    events = (Event * max(1, max_events))()
    pr = Problem(M=M, N=N, K=K, alpha=alpha, beta=beta, A=_ptr(A), lda=K, B=_ptr(B), ldb=N,
                 Cin=_ptr(Cin_a), ldc=N, out_dtype=OUT_F32 if out == "f32" else OUT_BF16,
                 acc_mode=ACC_FP64 if acc == "fp64" else ACC_FP32SEQ, Cout=_ptr(Cout),
                 tile_m=tile_m, tile_n=tile_n, bk=bk, u_acc=u_acc, lambda1=lambda1, lambda2=lambda2,
                 ft_level=ft_level, n_inj=len(inj), inj=C.cast(inj_arr, C.c_void_p),
                 counts=C.cast(C.pointer(counts), C.c_void_p),
                 events=C.cast(events, C.c_void_p), max_events=max_events, pad0=0,
                 P_out=_ptr(P), resid_row=_ptr(rr), resid_col=_ptr(rc), tau_row=_ptr(tr), tau_col=_ptr(tc),
                 ks=ks)
    err = lib().oracle_ftgemm(C.byref(pr))
    if err:
        raise ValueError(f"oracle_ftgemm error {err}")
    cnt = {n: getattr(counts, n) for n, _ in Counts._fields_}
    evs = []
    for i in range(min(cnt["events"], max_events)):
        e = events[i]
        evs.append(dict(row=e.row, col=e.col, tile_m=e.tile_m, tile_n=e.tile_n, kind=e.kind,
                        n_rows=e.n_rows, n_cols=e.n_cols, k_checked=e.k_checked, resid_row=e.resid_row,
                        resid_col=e.resid_col, tau_row=e.tau_row, tau_col=e.tau_col))
    evs.sort(key=lambda e: (e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"]))
    if out == "f32":
        Cv, bits = Cout, None
    else:
        bits = Cout
        Cv = (Cout.astype(np.uint32) << np.uint32(16)).view(np.float32)
    return Result(C=Cv, C_bits=bits, P=P, counts=cnt, events=evs,
                  resid_row=rr, resid_col=rc, tau_row=tr, tau_col=tc)


def encode_col(A, tile_m):
    A = _f32(A); M, K = A.shape
    out = np.zeros((-(-M // tile_m), K), dtype=np.float64)
    assert lib().oracle_encode_col(M, K, _ptr(A), K, tile_m, _ptr(out)) == 0
    return out


def encode_row(B, tile_n):
    B = _f32(B); K, N = B.shape
    out = np.zeros((-(-N // tile_n), K), dtype=np.float64)
    assert lib().oracle_encode_row(K, N, _ptr(B), N, tile_n, _ptr(out)) == 0
    return out


def gemm_f64(A, B, Cin=None, alpha=1.0, beta=0.0):
    A = _f32(A); B = _f32(B); M, K = A.shape; N = B.shape[1]
    Cin_a = _f32(Cin) if Cin is not None else None
    out = np.zeros((M, N), dtype=np.float64)
    assert lib().oracle_gemm_f64(M, N, K, alpha, _ptr(A), K, _ptr(B), N, beta, _ptr(Cin_a), N, _ptr(out)) == 0
    return out


def double_to_bf16(d: float) -> int:
    return int(lib().oracle_double_to_bf16(float(d)))


def num_threads() -> int:
    return int(lib().oracle_num_threads())
