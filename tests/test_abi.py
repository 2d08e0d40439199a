"""CPU-only checks of the C-ABI library: it builds/loads, exports every symbol that
include/codedinv.h declares, and rejects host-checkable bad arguments without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

import fixtures as fx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ci():
    from paper_2106_06445_b200 import build
    build.build()
    from paper_2106_06445_b200 import codedinv
    return codedinv


def declared_symbols(*headers):
    syms = set()
    for h in headers:
        syms |= set(re.findall(r"CI_API[^;(]*?\b(ci_\w+)\s*\(", open(os.path.join(ROOT, "include", h + ".h")).read()))
    return sorted(syms)


PRODUCT_HEADERS = ("codedinv", "codedinv_testing")


def test_header_declares_the_north_star_entry_points():
    syms = declared_symbols("codedinv")
    for name in ("ci_forward_h", "ci_inverse_h", "ci_encode", "ci_decode", "ci_classify",
                 "ci_serve_group"):
        assert name in syms


def test_library_exports_every_declared_symbol(ci):
    lib = ctypes.CDLL(ci.LIB_PATH)
    for name in declared_symbols(*PRODUCT_HEADERS):
        assert hasattr(lib, name), name
    assert sorted(ci.EXPORTS + ci.TESTING_EXPORTS) == declared_symbols(*PRODUCT_HEADERS)


def test_probe_library_is_separate(ci):
    """The tcgen05 probes (include/codedinv_probe.h) live in libcodedinv_probe.so only."""
    import subprocess
    from paper_2106_06445_b200 import build
    probe = ctypes.CDLL(build.PROBE_LIB)
    for name in declared_symbols("codedinv_probe"):
        assert hasattr(probe, name), name
    dyn = subprocess.run(["nm", "-D", "--defined-only", ci.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_symbols("codedinv_probe"):
        assert name not in dyn, name
    elf = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-text", ci.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "k_umma_gemm" not in elf and "k_umma_rate" not in elf


def test_library_is_sm100a(ci):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ci.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_host_side_argument_errors(ci):
    lib = ci._lib
    # bad arch -> synchronous error before any device work
    a = ci.to_ci_arch(fx.ARCH_T)
    a.n_stages = 0
    h = ctypes.c_void_p()
    p = np.zeros(4, np.float32)
    st = lib.ci_model_create(ctypes.byref(a), p.ctypes.data_as(ctypes.c_void_p), 4, 0, 0, ctypes.byref(h))
    assert st == ci.CI_ERR_INVALID_SHAPE and "arch" in ci.ci_last_error()
    # parameter count mismatch
    a = ci.to_ci_arch(fx.ARCH_T)
    st = lib.ci_model_create(ctypes.byref(a), p.ctypes.data_as(ctypes.c_void_p), 4, 0, 0, ctypes.byref(h))
    assert st == ci.CI_ERR_DIM_MISMATCH
    # unknown precision
    st = lib.ci_model_create(ctypes.byref(a), p.ctypes.data_as(ctypes.c_void_p), 4, 9, 0, ctypes.byref(h))
    assert st == ci.CI_ERR_INVALID_ARG
    # decode: k < 1, misaligned, null workspace
    assert lib.ci_decode(0, 1, 4, None, None, None, None, 0, None) == ci.CI_ERR_INVALID_ARG
    assert lib.ci_decode(2, -1, 4, None, None, None, None, 0, None) == ci.CI_ERR_INVALID_ARG
    buf = (ctypes.c_float * 64)()
    addr = ctypes.addressof(buf)
    assert lib.ci_decode(2, 1, 4, ctypes.c_void_p(addr), ctypes.c_void_p(addr + 32),
                         ctypes.c_void_p(addr), None, 0, None) == ci.CI_ERR_WORKSPACE
    # NULL model
    assert lib.ci_feature_dim(None) == -1
    assert lib.ci_forward_h(None, None, None, 1, None, 0, None) == ci.CI_ERR_INVALID_ARG
    assert lib.ci_make_drops(0, 1, 1, None, None) == ci.CI_ERR_INVALID_ARG


def test_binding_has_no_cpu_fallback():
    """The product package never imports the oracle (or numpy math for the path)."""
    pkg = os.path.join(ROOT, "paper_2106_06445_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in src.replace("no CPU fallback", ""), f


def test_hot_path_plans_have_specialised_kernels():
    """Every stage of the benchmarked archs (C3/C4: Arch C; C3R: the residual arch) in both
    tensor-core precisions must dispatch to a compile-time specialised stage kernel: a plan/spec
    mismatch (e.g. the SMEM-state flag) would silently fall back to the ~3x slower generic
    kernel.  Host-only planner query, no GPU needed."""
    from paper_2106_06445_b200 import codedinv as ci
    import fixtures as fx
    for arch, pms in ((fx.ARCH_C, (0, 1, 2)), (fx.ARCH_CR, (0, 2))):   # pm: bf16, f16x2, f16x3 (CI_PREC_FP32)
        for (C, H, W, c, m, nb) in arch.stage_shapes():
            for pm in pms:
                q = -c if arch.block == "residual" else c
                plan = ci.ci_test_plan(H, W, q, m, pm)
                assert plan["static"] == 1, (arch.name, H, c, m, pm, plan)
                assert plan["tmem_cols"] <= 512 and plan["smem"] <= 227 * 1024
    # Arch C: stage 1 on k_stage_ts, stage 2 on k_stage_ts2, stage 3 on the interleaved raster
    # (one tile of eight 4x4 images: Wp = 32), in every precision
    for pm in (0, 1, 2):
        assert ci.ci_test_plan(16, 16, 6, 64, pm)["ts"] == 1
        assert ci.ci_test_plan(8, 8, 24, 128, pm)["ts"] == 2
        p3 = ci.ci_test_plan(4, 4, 96, 256, pm)
        assert p3["nopad"] == 2 and p3["Wp"] == 32 and p3["T"] == 1 and p3["I"] == 8
    # C3R stage 1 in the contract precision: the wide-hst plan (conv2 as 3 x 16 = 48 columns over
    # the hidden map in shared memory, 5 tiles, state in SMEM)
    p1 = ci.ci_test_plan(16, 16, -12, 64, 2)
    assert p1["hst"] == 1 and p1["Nc2"] == 48 and p1["T"] == 5 and p1["static"] == 1
