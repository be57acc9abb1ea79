"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, exports
every symbol include/ftgemm.h declares, the host plan table is consistent, and
argument errors are reported synchronously (no device needed).  There is no
CPU fallback: on a machine without an sm_100 GPU a well-formed call fails with
FTGEMM_ERR_UNSUPPORTED."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ftgemm.h")


@pytest.fixture(scope="module")
def F():
    from paper_2305_01024_b200 import build
    build.build()
    from paper_2305_01024_b200 import ftgemm
    ftgemm.lib()
    return ftgemm


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"FTGEMM_API\s+[\w\s\*]+?\b(ftgemm_\w+)\s*\(", txt)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("ftgemm_plan", "ftgemm_encode", "ftgemm_run", "ftgemm_report", "ftgemm_report_reset",
              "ftgemm_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(F):
    lib = F.lib()
    for s in declared_symbols():
        assert hasattr(lib, s), s
    assert lib.ftgemm_version() == 2
    assert lib.ftgemm_device_arch() == 1000


def test_built_for_sm100a(F):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", F.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass      # tcgen05.mma
    assert "UTMALDG" in sass                           # TMA loads
    assert "LDTM" in sass                              # tcgen05.ld


def test_struct_layouts(F, tmp_path):
    """The ctypes mirrors in the binding have the header's sizes and offsets (compiled with gcc)."""
    import subprocess
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "ftgemm.h"\n'
                   'int main(){printf("%zu %zu %zu %zu %zu %zu\\n", sizeof(ftgemm_inject_t), sizeof(ftgemm_event_t),'
                   ' sizeof(ftgemm_counts_t), sizeof(ftgemm_plan_t), offsetof(ftgemm_plan_t, tiles_m),'
                   ' offsetof(ftgemm_plan_t, u_acc));return 0;}')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = list(map(int, subprocess.run([str(exe)], capture_output=True, text=True).stdout.split()))
    assert got == [C.sizeof(F.Inject), C.sizeof(F.Event), C.sizeof(F.Counts), C.sizeof(F.PlanStruct),
                   F.PlanStruct.tiles_m.offset, F.PlanStruct.u_acc.offset]
    assert got[:3] == [40, 56, 72]


@pytest.mark.parametrize("dtype", ["f32_simt", "tf32", "bf16"])
def test_plan_table(F, dtype):
    p = F.plan(dtype, 8192, 8192, 8192)
    if dtype == "f32_simt":
        assert (p.bm, p.bn, p.bk, p.check_tile_m, p.check_tile_n) == (128, 128, 32, 128, 128)
        assert p.u_acc == 2.0 ** -24
    else:
        assert (p.bm, p.bn) == (128, 256) and p.check_tile_m == 125 and p.check_tile_n == 252
        assert p.bk == (32 if dtype == "tf32" else 64)
        assert p.u_acc == 2.0 ** -23
    assert p.tiles_m == -(-8192 // p.check_tile_m) and p.tiles_n == -(-8192 // p.check_tile_n)
    assert 0 < p.enc_b_offset < p.enc_bytes and p.enc_b_offset + p.enc_b_bytes == p.enc_bytes
    assert p.report_bytes > 0 and p.max_events == 4096
    if dtype != "f32_simt":
        small = F.plan(dtype, 2048, 2048, 2048)          # too few 125 x 252 tiles for 2 waves
        assert small.bn == 128 and small.shape_class == 1 and small.cta_group == 1
        sm = F.plan(dtype, 128, 16384, 16384)             # skinny M: one CTA pair per unit
        assert sm.bn == 256 and sm.cta_group == 2 and sm.tiles_m == 2
        sn = F.plan(dtype, 16384, 128, 16384)             # skinny N: a single check-tile column
        assert sn.bn == 256 and sn.tiles_n == 1
        big = F.plan(dtype, 8192, 8192, 8192)
        assert big.cta_group == 2 and big.stages >= 4
        # wave-quantised class choice (profiles/r1d_tile_classes.md): 99 pair units
        # (2 waves) beat 330 BN=128 tiles (3 waves) at 8192 x 512 x 8192
        nar = F.plan(dtype, 8192, 512, 8192)
        assert nar.bn == 256 and nar.cta_group == 2
        k1 = F.plan(dtype, 8192, 8192, 1024)
        assert k1.bn == 256 and k1.cta_group == 2
        k128 = F.plan(dtype, 16384, 16384, 128)       # epilogue-bound: one CTA per MMA
        assert k128.cta_group == 1 and k128.bn == (128 if dtype == "tf32" else 256)
        k512 = F.plan(dtype, 8192, 8192, 512)         # TF32: the cost model from K = 512
        assert (k512.bn, k512.cta_group) == ((256, 2) if dtype == "tf32" else (256, 1))


def test_plan_errors(F):
    for dims in [(0, 8, 8), (8, -1, 8), (8, 8, 0)]:
        with pytest.raises(F.FtgemmError) as e:
            F.plan("bf16", *dims)
        assert e.value.code == 1
    with pytest.raises(F.FtgemmError) as e:
        F.plan(7, 8, 8, 8)
    assert e.value.code == 1


def test_synchronous_argument_errors(F):
    lib = F.lib()
    buf = (C.c_uint8 * 4096)()
    base = (C.addressof(buf) + 255) & ~255
    # null operands
    assert lib.ftgemm_run(2, 64, 64, 64, 1.0, None, 64, base, 64, 0.0, base, 64, None, 0, None, 0, None, None) == 1
    # leading dimension too small
    assert lib.ftgemm_run(2, 64, 64, 64, 1.0, base, 32, base, 64, 0.0, base, 64, None, 0, None, 0, None, None) == 1
    # FT without workspaces
    assert lib.ftgemm_run(2, 64, 64, 64, 1.0, base, 64, base, 64, 0.0, base, 64, None, 2, None, 0, None, None) == 1
    # misaligned base (TMA needs 16-byte bases)
    assert lib.ftgemm_run(2, 64, 64, 64, 1.0, base + 2, 64, base, 64, 0.0, base, 64, None, 0, None, 0, None, None) == 2
    # row pitch not a multiple of 16 bytes
    assert lib.ftgemm_run(2, 64, 64, 60, 1.0, base, 60, base, 64, 0.0, base, 64, None, 0, None, 0, None, None) == 2
    # bad encode selector
    assert lib.ftgemm_encode(2, 64, 64, 64, base, 64, base, 64, base, 4, None) == 1
    assert "which" in lib.ftgemm_last_error().decode()


def test_no_cpu_fallback(F):
    """A well-formed call on a host without an sm_100 device fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = F.lib()
    buf = (C.c_uint8 * (64 * 64 * 2 + 512))()
    base = (C.addressof(buf) + 255) & ~255
    rc = lib.ftgemm_run(2, 64, 64, 64, 1.0, base, 64, base, 64, 0.0, base, 64, None, 0, None, 0, None, None)
    assert rc == 2
    assert "sm_100" in lib.ftgemm_last_error().decode()


def test_cost_model_host(F):
    """ftgemm_cost_model (host-only) against the oracle's closed form and its
    pins (tests/test_oracle.py::test_cost_model_online_vs_offline)."""
    import math
    from oracle import cost_model as cm
    assert C.sizeof(F.Cost) == 40
    for g0, tiles in ((1 / 256, 64), (1e-6, 2048), (0.0, 5), (0.01, 10), (1e-3, 108900)):
        c = F.cost_model(g0, tiles)
        g = cm.gamma(g0, tiles)
        assert abs(c["gamma"] - g) <= 1e-12 * max(1.0, g) and c["online_expected_runs"] == 1.0
        if g < 0.5:
            assert abs(c["offline_expected_runs"] - cm.offline_expected_runs(g)) <= 1e-12 * cm.offline_expected_runs(g)
        else:
            assert math.isinf(c["offline_expected_runs"])
    c = F.cost_model(1 / 256, 64)
    assert abs(c["gamma"] - 0.221580) < 5e-7 and abs(c["offline_expected_runs"] - 1.397925) < 5e-7
    for bad in ((-0.1, 4), (1.0, 4), (0.1, 0)):
        with pytest.raises(F.FtgemmError) as e:
            F.cost_model(*bad)
        assert e.value.code == 1


def test_run_offline_argument_errors(F):
    lib = F.lib()
    out = (C.c_int32 * 2)()
    vp = C.c_void_p(16)
    # max_runs < 1, beta != 0 without a backup, inj_run outside [0, max_runs)
    assert lib.ftgemm_run_offline(2, 64, 64, 64, 1.0, vp, 64, vp, 64, 0.0, vp, 64, None, vp, None, None, 0, 0,
                                  vp, C.cast(out, C.c_void_p), None) == 1
    assert lib.ftgemm_run_offline(2, 64, 64, 64, 1.0, vp, 64, vp, 64, 0.5, vp, 64, None, vp, None, None, 0, 2,
                                  vp, C.cast(out, C.c_void_p), None) == 1
    inj = (F.Inject * 1)(F.Inject(0, 0, 0, 3, 0, 0, 0.0))
    run = (C.c_int32 * 1)(5)
    assert lib.ftgemm_run_offline(2, 64, 64, 64, 1.0, vp, 64, vp, 64, 0.0, vp, 64, None, vp, C.cast(inj, C.c_void_p),
                                  C.cast(run, C.c_void_p), 1, 2, vp, C.cast(out, C.c_void_p), None) == 1


def test_nonfused_host_checks(F):
    """Workspace query (host) and the synchronous argument checks of the
    non-fused baseline: TF32 is unsupported (cuBLAS rounds TF32 operands to
    nearest, the encode truncates as the tensor core does)."""
    b = F.nonfused_workspace("bf16", 1000, 1112, 704)
    assert b >= 1000 * 1112 * 4
    with pytest.raises(F.FtgemmError) as e:
        F.nonfused_workspace("tf32", 64, 64, 64)
    assert e.value.code == 2
    lib = F.lib()
    vp = C.c_void_p(16)
    assert lib.ftgemm_run_nonfused(1, 64, 64, 64, 1.0, vp, 64, vp, 64, 0.0, vp, 64, vp, vp, 2, None, 0, vp, None) == 2
    assert lib.ftgemm_run_nonfused(2, 64, 64, 64, 1.0, vp, 64, vp, 64, 0.0, vp, 64, None, None, 2, None, 0, vp, None) == 1


def test_explicit_tile_class(F):
    """An explicit class in the dtype code (FTGEMM_TILE(bn, cta_group)) fixes the
    tensor-core plan for that call only -- there is no process-wide state --
    and wins over every shape rule; plan.dtype is the plan's explicit code, so
    re-planning with it reproduces the plan (the multi-GPU partition runs every
    rank with the full problem's check tiles this way).  Invalid classes and a
    class on F32_SIMT are argument errors."""
    auto = F.plan("bf16", 8192, 8192, 8192)
    assert (auto.bn, auto.cta_group) == (256, 2)
    assert auto.dtype == F.tile_code("bf16", 256, 2) == (2 | 2 << 8 | 2 << 12)
    p = F.plan("bf16", 8192, 8192, 8192, tile=(128, 1))
    assert (p.bn, p.cta_group, p.check_tile_n) == (128, 1, 124)
    assert F.plan(p.dtype, 8192, 8192, 8192) == p
    assert F.plan("bf16", 8192, 8192, 8192) == auto            # nothing ambient changed
    sn = F.plan("bf16", 16384, 128, 16384)
    assert sn.bn == 256 and sn.tiles_n == 1
    sn2 = F.plan("bf16", 16384, 128, 16384, tile=(128, 2))
    assert (sn2.bn, sn2.cta_group, sn2.tiles_n) == (128, 2, 2)
    s = F.plan("f32_simt", 1024, 1024, 1024)
    assert s.bn == 128 and s.check_tile_n == 128 and s.dtype == F.F32_SIMT
    for bad in ((192, 1), (256, 3)):
        with pytest.raises(F.FtgemmError) as e:
            F.plan("bf16", 64, 64, 64, tile=bad)
        assert e.value.code == 1
    for code in (F.tile_code("f32_simt", 128, 1), F.BF16 | (1 << 8), F.BF16 | (1 << 20)):
        with pytest.raises(F.FtgemmError) as e:
            F.plan(code, 64, 64, 64)
        assert e.value.code == 1
    # encode and run with different codes must not be mixed: the layouts differ
    a, b = F.encode_layout(auto.dtype, 8192, 8192, 8192), F.encode_layout(p.dtype, 8192, 8192, 8192)
    assert a["bt_ld"] == 33 * 256 and b["bt_ld"] == 67 * 128
