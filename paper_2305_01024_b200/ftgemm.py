"""Thin Python binding of libftgemm (include/ftgemm.h) — argument marshalling only.

Every step of the path runs in the CUDA kernels behind the C ABI; this module
converts torch tensors to device pointers / sizes / streams and ctypes structs
back to Python objects.  There is no CPU fallback: if the shared library is
missing or the device is not an sm_100 GPU, calls raise.

PyTorch is used only for device memory (the workspaces are torch tensors) and
streams (torch.cuda.current_stream()).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FTGEMM_LIB") or os.path.join(_HERE, "libftgemm.so")   # FTGEMM_LIB: development variants

F32_SIMT, TF32, BF16 = 0, 1, 2
DTYPES = {"f32_simt": F32_SIMT, "tf32": TF32, "bf16": BF16}
FT_OFF, FT_DETECT, FT_CORRECT, FT_DETECT_ROWS = 0, 1, 2, 3
INJ_FLIP, INJ_ADD = 0, 1
TGT_ACC, TGT_ROW_REF, TGT_COL_REF = 0, 1, 2
EV_CORRECTED, EV_CHECKSUM_ONLY, EV_UNCORRECTABLE, EV_LOCATED, EV_DETECTED = 1, 2, 3, 4, 5
ERR = {0: "OK", 1: "INVALID_VALUE", 2: "UNSUPPORTED", 3: "CUDA"}


class Inject(C.Structure):
    _fields_ = [("row", C.c_int64), ("col", C.c_int64), ("k_elem", C.c_int64),
                ("bit", C.c_int32), ("mode", C.c_int32), ("target", C.c_int32), ("addend", C.c_float)]


class Event(C.Structure):
    _fields_ = [("row", C.c_int64), ("col", C.c_int64), ("tile_m", C.c_int32), ("tile_n", C.c_int32),
                ("kind", C.c_int32), ("n_rows", C.c_int32), ("n_cols", C.c_int32), ("k_checked", C.c_int32),
                ("resid_row", C.c_float), ("resid_col", C.c_float), ("tau_row", C.c_float), ("tau_col", C.c_float)]


class Counts(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("tiles_checked", "tiles_detected", "corrected", "checksum_only",
                                         "uncorrectable", "located", "events", "dropped")] + \
               [("max_resid_ratio", C.c_float), ("pad", C.c_int32)]


class PlanStruct(C.Structure):
    _fields_ = [("dtype", C.c_int32), ("shape_class", C.c_int32), ("bm", C.c_int32), ("bn", C.c_int32),
                ("bk", C.c_int32), ("check_tile_m", C.c_int32), ("check_tile_n", C.c_int32),
                ("off_tile_m", C.c_int32), ("off_tile_n", C.c_int32), ("stages", C.c_int32),
                ("cta_group", C.c_int32), ("max_events", C.c_int32), ("max_inject", C.c_int32),
                ("pad0", C.c_int32), ("tiles_m", C.c_int64), ("tiles_n", C.c_int64), ("enc_bytes", C.c_int64),
                ("enc_b_offset", C.c_int64), ("enc_b_bytes", C.c_int64), ("report_bytes", C.c_int64),
                ("u_acc", C.c_float), ("lambda1", C.c_float), ("lambda2", C.c_float), ("pad1", C.c_int32)]


class EncLayoutStruct(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("ac", "br", "bt", "rownorm", "colnorm", "acnorm", "brnorm", "kp", "bt_ld", "y")]


class Cost(C.Structure):
    _fields_ = [("gamma0", C.c_double), ("tiles", C.c_int64), ("gamma", C.c_double),
                ("online_expected_runs", C.c_double), ("offline_expected_runs", C.c_double)]


SYMBOLS = ("ftgemm_plan", "ftgemm_encode", "ftgemm_encode_layout", "ftgemm_run", "ftgemm_run_fused", "ftgemm_run_online", "ftgemm_run_offline", "ftgemm_cost_model",
           "ftgemm_nonfused_workspace", "ftgemm_run_nonfused",
           "ftgemm_report", "ftgemm_report_reset", "ftgemm_last_error", "ftgemm_version", "ftgemm_device_arch",
           "ftgemm_plan_batched", "ftgemm_encode_batched", "ftgemm_run_batched")
DTYPE_MASK = 0xFF


def tile_code(dtype, bn: int, cta_group: int) -> int:
    """dtype code with an explicit tensor-core tile class (FTGEMM_TILE in include/ftgemm.h)."""
    tb = bn // 128 if bn in (128, 256) else 0xF           # anything else: rejected by the library
    return _dt(dtype) | (tb << 8) | ((cta_group & 0xF) << 12)

_lib = None


def lib():
    """Load libftgemm.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2305_01024_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        i64, i32, vp = C.c_int64, C.c_int32, C.c_void_p
        L.ftgemm_plan.argtypes = [C.c_int, i64, i64, i64, C.POINTER(PlanStruct)]
        L.ftgemm_encode.argtypes = [C.c_int, i64, i64, i64, vp, i64, vp, i64, vp, C.c_int, vp]
        L.ftgemm_encode_layout.argtypes = [C.c_int, i64, i64, i64, C.POINTER(EncLayoutStruct)]
        L.ftgemm_run.argtypes = [C.c_int, i64, i64, i64, C.c_float, vp, i64, vp, i64, C.c_float, vp, i64,
                                 vp, C.c_int, vp, i32, vp, vp]
        L.ftgemm_run_fused.argtypes = L.ftgemm_run.argtypes
        L.ftgemm_run_online.argtypes = [C.c_int, i64, i64, i64, C.c_float, vp, i64, vp, i64, C.c_float, vp, i64,
                                        vp, C.c_int, i64, vp, i32, vp, vp]
        L.ftgemm_run_offline.argtypes = [C.c_int, i64, i64, i64, C.c_float, vp, i64, vp, i64, C.c_float, vp, i64,
                                         vp, vp, vp, vp, i32, i32, vp, vp, vp]
        L.ftgemm_cost_model.argtypes = [C.c_double, i64, C.POINTER(Cost)]
        L.ftgemm_nonfused_workspace.argtypes = [C.c_int, i64, i64, i64, C.POINTER(C.c_int64)]
        L.ftgemm_run_nonfused.argtypes = [C.c_int, i64, i64, i64, C.c_float, vp, i64, vp, i64, C.c_float, vp, i64,
                                          vp, vp, C.c_int, vp, i32, vp, vp]
        L.ftgemm_report.argtypes = [vp, C.POINTER(Counts), vp, i32, vp]
        L.ftgemm_plan_batched.argtypes = [C.c_int, i64, i64, i64, i64, C.POINTER(PlanStruct)]
        L.ftgemm_encode_batched.argtypes = [C.c_int, i64, i64, i64, i64, vp, i64, i64, vp, i64, i64, vp, i64, C.c_int, vp]
        L.ftgemm_run_batched.argtypes = [C.c_int, i64, i64, i64, i64, C.c_float, vp, i64, i64, vp, i64, i64, C.c_float,
                                         vp, i64, i64, vp, i64, C.c_int, vp, i32, vp, vp]
        L.ftgemm_report_reset.argtypes = [vp, i64, vp]
        L.ftgemm_last_error.restype = C.c_char_p
        for n in SYMBOLS:
            if n != "ftgemm_last_error" and hasattr(L, n):
                getattr(L, n).restype = C.c_int
        _lib = L
    return _lib


class FtgemmError(RuntimeError):
    def __init__(self, code: int, where: str):
        msg = lib().ftgemm_last_error().decode()
        super().__init__(f"{where}: {ERR.get(code, code)}: {msg}")
        self.code = code


def _check(code: int, where: str):
    if code != 0:
        raise FtgemmError(code, where)


def _dt(dtype) -> int:
    return DTYPES[dtype] if isinstance(dtype, str) else int(dtype)


_TORCH_DT = {F32_SIMT: torch.float32, TF32: torch.float32, BF16: torch.bfloat16}


def _operand(name: str, t: torch.Tensor, dtype, rows: int | None = None, cols: int | None = None):
    """Argument checks the C ABI cannot make (it sees only pointers): a CUDA
    tensor of the dtype's operand type, 2-D, unit inner stride, given shape."""
    want = _TORCH_DT[_dt(dtype) & DTYPE_MASK]
    if not isinstance(t, torch.Tensor) or t.dim() != 2:
        raise ValueError(f"{name}: expected a 2-D torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor (there is no CPU path)")
    if t.dtype != want:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {want}")
    if t.stride(1) != 1 or t.stride(0) < t.shape[1]:
        raise ValueError(f"{name}: rows must be contiguous (stride(1) == 1, stride(0) >= cols)")
    if (rows is not None and t.shape[0] != rows) or (cols is not None and t.shape[1] != cols):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected ({rows}, {cols})")


def _gemm_operands(dtype, A, B, C_):
    _operand("A", A, dtype)
    M, K = A.shape
    _operand("B", B, dtype, rows=K)
    N = B.shape[1]
    _operand("C", C_, dtype, rows=M, cols=N)
    return M, N, K


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


@dataclass
class Plan:
    dtype: int
    shape_class: int
    bm: int
    bn: int
    bk: int
    check_tile_m: int
    check_tile_n: int
    off_tile_m: int
    off_tile_n: int
    stages: int
    cta_group: int
    max_events: int
    max_inject: int
    tiles_m: int
    tiles_n: int
    enc_bytes: int
    enc_b_offset: int
    enc_b_bytes: int
    report_bytes: int
    u_acc: float
    lambda1: float
    lambda2: float


def plan(dtype, M: int, N: int, K: int, tile: tuple[int, int] | None = None) -> Plan:
    """tile = (bn, cta_group): an explicit tensor-core tile class; plan.dtype is the
    plan's fully explicit dtype code (pass it to encode / run)."""
    if tile is not None:
        dtype = tile_code(dtype, *tile)
    p = PlanStruct()
    _check(lib().ftgemm_plan(_dt(dtype), M, N, K, C.byref(p)), "ftgemm_plan")
    return Plan(**{f: getattr(p, f) for f in Plan.__dataclass_fields__})


def encode_layout(dtype, M: int, N: int, K: int) -> dict:
    """Byte offsets of the encode results inside enc_ws (ftgemm_encode_layout)."""
    e = EncLayoutStruct()
    _check(lib().ftgemm_encode_layout(_dt(dtype), M, N, K, C.byref(e)), "ftgemm_encode_layout")
    return {f: getattr(e, f) for f, _ in EncLayoutStruct._fields_}


def alloc_workspaces(pl: Plan, device="cuda"):
    """enc_ws and report_ws as torch device tensors (PyTorch owns device memory)."""
    enc = torch.empty(max(pl.enc_bytes, 256), dtype=torch.uint8, device=device)
    rep = torch.zeros(pl.report_bytes, dtype=torch.uint8, device=device)
    return enc, rep


def encode(dtype, A: torch.Tensor | None, B: torch.Tensor | None, enc_ws: torch.Tensor, *, M: int, N: int, K: int,
           which: int = 3, stream=None):
    if which & 1:
        _operand("A", A, dtype, rows=M, cols=K)
    if which & 2:
        _operand("B", B, dtype, rows=K, cols=N)
    if enc_ws.numel() < plan(dtype, M, N, K).enc_bytes:
        raise ValueError("enc_ws smaller than plan.enc_bytes")
    _check(lib().ftgemm_encode(_dt(dtype), M, N, K,
                               A.data_ptr() if A is not None else None, A.stride(0) if A is not None else K,
                               B.data_ptr() if B is not None else None, B.stride(0) if B is not None else N,
                               enc_ws.data_ptr(), which, _stream(stream)), "ftgemm_encode")


def _inj_array(injections):
    inj = list(injections or ())
    if not inj:
        return None, 0
    arr = (Inject * len(inj))()
    for i, x in enumerate(inj):
        if isinstance(x, dict):
            x = (x["row"], x["col"], x["k_elem"], x.get("bit", 0), x.get("mode", INJ_FLIP),
                 x.get("target", TGT_ACC), x.get("addend", 0.0))
        arr[i] = Inject(*x)
    return arr, len(inj)


def run(dtype, A: torch.Tensor, B: torch.Tensor, C_: torch.Tensor, *, alpha: float = 1.0, beta: float = 0.0,
        enc_ws: torch.Tensor | None = None, ft_level: int = FT_CORRECT, injections=(),
        report_ws: torch.Tensor | None = None, stream=None, fuse_a: bool = False):
    """fuse_a: the A-side encode runs inside the GEMM kernel (ftgemm_run_fused);
    enc_ws then needs only the B part."""
    M, N, K = _gemm_operands(dtype, A, B, C_)
    arr, n = _inj_array(injections)
    fn = lib().ftgemm_run_fused if fuse_a else lib().ftgemm_run
    _check(fn(_dt(dtype), M, N, K, alpha, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                            beta, C_.data_ptr(), C_.stride(0),
                            enc_ws.data_ptr() if enc_ws is not None else None, ft_level,
                            C.cast(arr, C.c_void_p) if arr is not None else None, n,
                            report_ws.data_ptr() if report_ws is not None else None, _stream(stream)),
           "ftgemm_run_fused" if fuse_a else "ftgemm_run")


def run_offline(dtype, A: torch.Tensor, B: torch.Tensor, C_: torch.Tensor, *, alpha: float = 1.0,
                beta: float = 0.0, enc_ws: torch.Tensor, report_ws: torch.Tensor, injections=(), inj_run=None,
                max_runs: int = 4, c_backup: torch.Tensor | None = None, stream=None):
    """Offline (detect-only) ABFT with re-computation.
    Returns (executions, clean).  inj_run[i]: the execution fault i strikes."""
    M, N, K = _gemm_operands(dtype, A, B, C_)
    arr, n = _inj_array(injections)
    runs = None
    if inj_run is not None:
        runs = (C.c_int32 * max(1, n))(*inj_run)
    if beta != 0.0 and c_backup is None:
        c_backup = torch.empty_like(C_)
    out = (C.c_int32 * 2)()
    _check(lib().ftgemm_run_offline(_dt(dtype), M, N, K, alpha, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                                    beta, C_.data_ptr(), C_.stride(0),
                                    c_backup.data_ptr() if c_backup is not None else None, enc_ws.data_ptr(),
                                    C.cast(arr, C.c_void_p) if arr is not None else None,
                                    C.cast(runs, C.c_void_p) if runs is not None else None, n, max_runs,
                                    report_ws.data_ptr(), C.cast(out, C.c_void_p), _stream(stream)),
           "ftgemm_run_offline")
    return int(out[0]), bool(out[1])


def nonfused_workspace(dtype, M: int, N: int, K: int) -> int:
    b = C.c_int64()
    _check(lib().ftgemm_nonfused_workspace(_dt(dtype), M, N, K, C.byref(b)), "ftgemm_nonfused_workspace")
    return int(b.value)


def run_nonfused(dtype, A: torch.Tensor, B: torch.Tensor, C_: torch.Tensor, *, alpha: float = 1.0, beta: float = 0.0,
                 enc_ws: torch.Tensor | None = None, nf_ws: torch.Tensor | None = None, ft_level: int = FT_CORRECT,
                 injections=(), report_ws: torch.Tensor | None = None, stream=None):
    """The non-fused ABFT baseline (cuBLAS GEMMs + separate verification kernel)."""
    M, N, K = _gemm_operands(dtype, A, B, C_)
    arr, n = _inj_array(injections)
    _check(lib().ftgemm_run_nonfused(_dt(dtype), M, N, K, alpha, A.data_ptr(), A.stride(0), B.data_ptr(),
                                     B.stride(0), beta, C_.data_ptr(), C_.stride(0),
                                     enc_ws.data_ptr() if enc_ws is not None else None,
                                     nf_ws.data_ptr() if nf_ws is not None else None, ft_level,
                                     C.cast(arr, C.c_void_p) if arr is not None else None, n,
                                     report_ws.data_ptr() if report_ws is not None else None, _stream(stream)),
           "ftgemm_run_nonfused")


def cost_model(gamma0: float, tiles: int) -> dict:
    """Online vs offline expected executions (host-only)."""
    c = Cost()
    _check(lib().ftgemm_cost_model(gamma0, tiles, C.byref(c)), "ftgemm_cost_model")
    return {f: getattr(c, f) for f, _ in Cost._fields_}


def run_online(dtype, A: torch.Tensor, B: torch.Tensor, C_: torch.Tensor, *, ks: int, alpha: float = 1.0,
               beta: float = 0.0, enc_ws: torch.Tensor, ft_level: int = FT_CORRECT, injections=(),
               report_ws: torch.Tensor, stream=None):
    """Online ABFT verified after every ks of K."""
    M, N, K = _gemm_operands(dtype, A, B, C_)
    arr, n = _inj_array(injections)
    _check(lib().ftgemm_run_online(_dt(dtype), M, N, K, alpha, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                                   beta, C_.data_ptr(), C_.stride(0), enc_ws.data_ptr(), ft_level, ks,
                                   C.cast(arr, C.c_void_p) if arr is not None else None, n, report_ws.data_ptr(),
                                   _stream(stream)), "ftgemm_run_online")


def report(report_ws: torch.Tensor, max_events: int = 4096, stream=None):
    cnt = Counts()
    evs = (Event * max(1, max_events))()
    _check(lib().ftgemm_report(report_ws.data_ptr(), C.byref(cnt), C.cast(evs, C.c_void_p), max_events,
                               _stream(stream)), "ftgemm_report")
    counts = {f: getattr(cnt, f) for f, _ in Counts._fields_ if f != "pad"}
    out = []
    for i in range(min(counts["events"], max_events)):
        e = evs[i]
        out.append(dict(row=e.row, col=e.col, tile_m=e.tile_m, tile_n=e.tile_n, kind=e.kind, n_rows=e.n_rows,
                        n_cols=e.n_cols, k_checked=e.k_checked, resid_row=e.resid_row, resid_col=e.resid_col, tau_row=e.tau_row,
                        tau_col=e.tau_col))
    out.sort(key=lambda e: (e["tile_m"], e["tile_n"], e["kind"], e["row"], e["col"]))
    return counts, out


def report_reset(report_ws: torch.Tensor, stream=None):
    _check(lib().ftgemm_report_reset(report_ws.data_ptr(), report_ws.numel(), _stream(stream)), "ftgemm_report_reset")


class FTGemm:
    """Convenience object: plan + workspaces for one (dtype, M, N, K).

    g = FTGemm("bf16", M, N, K); g.encode(A, B); g.run(A, B, C); counts, events = g.report()

    tile = (bn, cta_group) fixes the tensor-core tile class (default: the plan's
    choice).  Every call passes the plan's explicit dtype code, so the encode and
    the run always agree on the layout of enc_ws.  With FT on, run() multiplies
    by the copy of B inside enc_ws: re-encode B (which=2) after changing it.
    """

    def __init__(self, dtype, M: int, N: int, K: int, device="cuda", tile: tuple[int, int] | None = None):
        self.M, self.N, self.K = M, N, K
        self.plan = plan(dtype, M, N, K, tile=tile)
        self.dtype = self.plan.dtype                 # explicit code: dtype | tile class
        self.enc_ws, self.report_ws = alloc_workspaces(self.plan, device)

    def _shape(self, A, B, C_=None):
        for name, t, want in (("A", A, (self.M, self.K)), ("B", B, (self.K, self.N)), ("C", C_, (self.M, self.N))):
            if t is not None and tuple(t.shape) != want:
                raise ValueError(f"{name} shape {tuple(t.shape)} != {want} of this FTGemm")

    def encode(self, A=None, B=None, which: int = 3, stream=None):
        self._shape(A, B)
        encode(self.dtype, A, B, self.enc_ws, M=self.M, N=self.N, K=self.K, which=which, stream=stream)

    def run(self, A, B, C_, *, alpha=1.0, beta=0.0, ft_level=FT_CORRECT, injections=(), stream=None, fuse_a=False):
        self._shape(A, B, C_)
        run(self.dtype, A, B, C_, alpha=alpha, beta=beta, enc_ws=self.enc_ws, ft_level=ft_level,
            injections=injections, report_ws=self.report_ws, stream=stream, fuse_a=fuse_a)

    def run_online(self, A, B, C_, *, ks, alpha=1.0, beta=0.0, ft_level=FT_CORRECT, injections=(), stream=None):
        self._shape(A, B, C_)
        run_online(self.dtype, A, B, C_, ks=ks, alpha=alpha, beta=beta, enc_ws=self.enc_ws, ft_level=ft_level,
                   injections=injections, report_ws=self.report_ws, stream=stream)

    def run_offline(self, A, B, C_, *, alpha=1.0, beta=0.0, injections=(), inj_run=None, max_runs=4,
                    c_backup=None, stream=None):
        self._shape(A, B, C_)
        return run_offline(self.dtype, A, B, C_, alpha=alpha, beta=beta, enc_ws=self.enc_ws,
                           report_ws=self.report_ws, injections=injections, inj_run=inj_run, max_runs=max_runs,
                           c_backup=c_backup, stream=stream)

    def run_nonfused(self, A, B, C_, *, alpha=1.0, beta=0.0, ft_level=FT_CORRECT, injections=(), stream=None):
        """Non-fused baseline; encode first with encode(A, B, which=3 | 4)."""
        self._shape(A, B, C_)
        if getattr(self, "nf_ws", None) is None:
            self.nf_ws = torch.empty(max(256, nonfused_workspace(self.dtype, self.M, self.N, self.K)),
                                     dtype=torch.uint8, device=self.enc_ws.device)
        run_nonfused(self.dtype, A, B, C_, alpha=alpha, beta=beta, enc_ws=self.enc_ws, nf_ws=self.nf_ws,
                     ft_level=ft_level, injections=injections, report_ws=self.report_ws, stream=stream)

    def __call__(self, A, B, C_=None, **kw):
        if C_ is None:
            C_ = torch.empty(self.M, self.N, dtype=A.dtype, device=A.device)
        if kw.get("ft_level", FT_CORRECT) != FT_OFF:
            self.encode(A, B, stream=kw.get("stream"))
        self.run(A, B, C_, **kw)
        return C_

    def report(self, max_events: int = 4096, stream=None):
        return report(self.report_ws, max_events, stream)

    def reset(self, stream=None):
        report_reset(self.report_ws, stream)

    @property
    def enc_b(self) -> torch.Tensor:
        """The B part of enc_ws (the unit broadcast with B across ranks)."""
        p = self.plan
        return self.enc_ws[p.enc_b_offset:p.enc_b_offset + p.enc_b_bytes]

    @property
    def enc_a(self) -> torch.Tensor:
        return self.enc_ws[:self.plan.enc_b_offset]


# ------------------------------------------------------------------ batched ---
def plan_batched(dtype, batch: int, M: int, N: int, K: int, tile: tuple[int, int] | None = None) -> Plan:
    if tile is not None:
        dtype = tile_code(dtype, *tile)
    p = PlanStruct()
    _check(lib().ftgemm_plan_batched(_dt(dtype), batch, M, N, K, C.byref(p)), "ftgemm_plan_batched")
    return Plan(**{f: getattr(p, f) for f in Plan.__dataclass_fields__})


def _batch_operand(name, t, dtype, batch, rows, cols):
    """A 3-D CUDA tensor [batch, rows, cols] with contiguous rows (stride(2) == 1)."""
    want = _TORCH_DT[_dt(dtype) & DTYPE_MASK]
    if not isinstance(t, torch.Tensor) or t.dim() != 3 or not t.is_cuda or t.dtype != want:
        raise ValueError(f"{name}: expected a 3-D CUDA tensor of {want}")
    if tuple(t.shape) != (batch, rows, cols):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {(batch, rows, cols)}")
    if t.stride(2) != 1 or t.stride(1) < cols:
        raise ValueError(f"{name}: rows must be contiguous")


class FTGemmBatched:
    """`batch` independent (M, N, K) problems in one persistent launch
    (ftgemm_run_batched).  A: [batch, M, K], B: [batch, K, N] (a stride-0
    expand of one B is allowed), C: [batch, M, N]; one encode workspace per
    problem in a single buffer."""

    def __init__(self, dtype, batch: int, M: int, N: int, K: int, device="cuda", tile: tuple[int, int] | None = None):
        self.batch, self.M, self.N, self.K = batch, M, N, K
        self.plan = plan_batched(dtype, batch, M, N, K, tile=tile)
        self.dtype = self.plan.dtype
        self.enc_stride = (self.plan.enc_bytes + 255) // 256 * 256
        self.enc_ws = torch.empty(self.enc_stride * batch, dtype=torch.uint8, device=device)
        self.report_ws = torch.zeros(self.plan.report_bytes, dtype=torch.uint8, device=device)

    def encode(self, A=None, B=None, which: int = 3, stream=None):
        if which & 1:
            _batch_operand("A", A, self.dtype, self.batch, self.M, self.K)
        if which & 2:
            _batch_operand("B", B, self.dtype, self.batch, self.K, self.N)
        _check(lib().ftgemm_encode_batched(
            self.dtype, self.batch, self.M, self.N, self.K,
            A.data_ptr() if A is not None else None, A.stride(1) if A is not None else self.K,
            A.stride(0) if A is not None else 0,
            B.data_ptr() if B is not None else None, B.stride(1) if B is not None else self.N,
            B.stride(0) if B is not None else 0,
            self.enc_ws.data_ptr(), self.enc_stride, which, _stream(stream)), "ftgemm_encode_batched")

    def run(self, A, B, C_, *, alpha=1.0, beta=0.0, ft_level=FT_CORRECT, injections=(), stream=None):
        _batch_operand("A", A, self.dtype, self.batch, self.M, self.K)
        _batch_operand("B", B, self.dtype, self.batch, self.K, self.N)
        _batch_operand("C", C_, self.dtype, self.batch, self.M, self.N)
        arr, n = _inj_array(injections)
        _check(lib().ftgemm_run_batched(
            self.dtype, self.batch, self.M, self.N, self.K, alpha, A.data_ptr(), A.stride(1), A.stride(0),
            B.data_ptr(), B.stride(1), B.stride(0), beta, C_.data_ptr(), C_.stride(1), C_.stride(0),
            self.enc_ws.data_ptr(), self.enc_stride, ft_level, C.cast(arr, C.c_void_p) if arr is not None else None,
            n, self.report_ws.data_ptr(), _stream(stream)), "ftgemm_run_batched")

    def report(self, max_events: int = 4096, stream=None):
        return report(self.report_ws, max_events, stream)

    def reset(self, stream=None):
        report_reset(self.report_ws, stream)
