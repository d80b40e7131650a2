"""CPU-only checks of the C ABI boundary: the library loads, exports every
symbol include/ss.h declares, and rejects invalid arguments with the documented
status BEFORE touching CUDA (so these run without a GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ss():
    import paper_2305_16513_b200 as ss
    return ss


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "ss.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_paper_entry_points():
    syms = declared_symbols()
    for s in ("ss_pool_sum", "ss_pool_max", "ss_conv1d", "ss_pool2d", "ss_out_len",
              "ss_status_string", "ss_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol(ss):
    out = subprocess.check_output(["nm", "-D", "--defined-only", ss.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (ss_[a-z0-9_]+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(ss.lib, s)
    assert set(ss.EXPORTED) == set(declared_symbols())


def test_library_is_sm100a(ss):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ss.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_abi_version_and_out_len(ss):
    assert ss.ss_abi_version() == 13
    assert ss.ss_out_len(10, 3, 1) == 8
    assert ss.ss_out_len(10, 3, 4) == 2
    assert ss.ss_out_len(2 ** 32, 31, 1) == 2 ** 32 - 30
    assert ss.ss_out_len(3, 4, 1) == -1
    assert ss.ss_out_len(0, 1, 1) == -1
    assert ss.ss_out_len(5, 0, 1) == -1
    assert ss.ss_out_len(5, 1, 0) == -1


FAKE_X = 0x10000000
FAKE_Y = 0x20000000


@pytest.mark.parametrize("fn", ["ss_pool_sum", "ss_pool_max"])
def test_pool_validation(ss, fn):
    f = getattr(ss, fn)
    assert f(0, FAKE_Y, 10, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_NULL
    assert f(FAKE_X, 0, 10, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_NULL
    assert f(FAKE_X, FAKE_Y, 0, 1, 1, 1, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert f(FAKE_X, FAKE_Y, 10, 0, 3, 1, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert f(FAKE_X, FAKE_Y, 10, 1, 0, 1, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert f(FAKE_X, FAKE_Y, 10, 1, 3, 0, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert f(FAKE_X, FAKE_Y, 10, 1, 11, 1, ss.SS_F32) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert "window exceeds input" in ss.ss_last_error()
    assert f(FAKE_X, FAKE_Y, 10, 1, 3, 1, 7) == ss.SS_ERR_UNSUPPORTED
    assert f(FAKE_X, FAKE_X + 8, 10, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_OVERLAP
    assert f(FAKE_X, FAKE_Y, 2 ** 62, 4, 3, 1, ss.SS_F32) == ss.SS_ERR_BAD_SIZE


def test_conv_validation(ss):
    f = [1.0, 2.0, 3.0]
    assert ss.ss_conv1d(FAKE_X, FAKE_Y, 10, 1, None, 3, 1) == ss.SS_ERR_NULL
    assert ss.ss_conv1d(0, FAKE_Y, 10, 1, f, 3, 1) == ss.SS_ERR_NULL
    assert ss.ss_conv1d(FAKE_X, FAKE_Y, 2, 1, f, 3, 1) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv1d(FAKE_X, FAKE_Y, 10, 1, f, 3, 1, ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    big = [0.0] * (ss.SS_K_MAX + 1)
    assert ss.ss_conv1d(FAKE_X, FAKE_Y, 5000, 1, big, len(big), 1) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_conv1d(FAKE_X, FAKE_Y, 10, 1, f, 0, 1) == ss.SS_ERR_BAD_SIZE


def test_pool2d_validation(ss):
    assert ss.ss_pool2d(0, FAKE_Y, 1, 8, 8, 2, 2, 2, 2, ss.SS_POOL_MAX) == ss.SS_ERR_NULL
    assert ss.ss_pool2d(FAKE_X, FAKE_Y, 0, 8, 8, 2, 2, 2, 2, ss.SS_POOL_MAX) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool2d(FAKE_X, FAKE_Y, 1, 8, 8, 9, 2, 1, 1, ss.SS_POOL_MAX) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_pool2d(FAKE_X, FAKE_Y, 1, 8, 8, 2, 2, 1, 1, 5) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_pool2d(FAKE_X, FAKE_Y, 1, 8, 8, 2, 2, 1, 1, ss.SS_POOL_AVG, ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_pool2d(FAKE_X + 2, FAKE_Y, 1, 8, 8, 2, 2, 1, 1, ss.SS_POOL_AVG) == ss.SS_ERR_BAD_SIZE


def test_status_strings(ss):
    for code in range(7):
        assert ss.ss_status_string(code).startswith("SS_")
    import torch
    if not torch.cuda.is_available():  # nothing was launched on a CPU box (a GPU session may have launched)
        assert ss.ss_launch_count() == 0


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2305_16513_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, fn)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", src).lower().replace("oracle_", "x"), fn


def test_window_spec_validation(ss):
    assert ss.ss_out_len_ex(10, 3, 1, 1, 0, 0) == 8
    assert ss.ss_out_len_ex(10, 3, 1, 2, 0, 0) == 6
    assert ss.ss_out_len_ex(3, 2, 1, 1, 1, 1) == 4
    assert ss.ss_out_len_ex(3, 4, 1, 2, 1, 1) == -1
    assert ss.ss_out_len_ex(3, 4, 1, 1, 0, 0) == -1
    assert ss.ss_out_len_ex(10, 3, 1, 0, 0, 0) == -1
    Z = ss.SS_PAD_ZEROS
    assert ss.ss_pool_sum_ex(FAKE_X, FAKE_Y, 10, 1, 3, 1, 0, 0, 0, Z, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_max_ex(FAKE_X, FAKE_Y, 10, 1, 3, 1, 1, -2, 0, Z, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_max_ex(FAKE_X, FAKE_Y, 3, 1, 3, 1, 2, 0, 0, Z, ss.SS_F32) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv1d_ex(FAKE_X, FAKE_Y, 10, 1, None, 3, 1, 1, 0, 0, Z, ss.SS_F32) == ss.SS_ERR_NULL
    assert ss.ss_conv1d_ex(FAKE_X, FAKE_Y, 10, 1, [1.0] * 3, 3, 1, 1, 0, 0, Z, ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    # padding modes: one reflection (pads <= N-1) / one period (<= N); unknown mode
    assert ss.ss_pool_min_ex(FAKE_X, FAKE_Y, 10, 1, 3, 1, 1, 10, 0, ss.SS_PAD_REFLECT, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_sum_ex(FAKE_X, FAKE_Y, 10, 1, 3, 1, 1, 0, 11, ss.SS_PAD_CIRCULAR, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_sum_ex(FAKE_X, FAKE_Y, 10, 1, 3, 1, 1, 1, 1, 9, ss.SS_F32) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_pool_min(0, FAKE_Y, 10, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_NULL
    assert ss.ss_pool_min(FAKE_X, FAKE_Y, 10, 1, 11, 1, ss.SS_F32) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT


def test_affine_window_validation(ss):
    f = ss.ss_affine_window
    X, Y, U, V = FAKE_X, FAKE_X + 0x1000000, FAKE_Y, FAKE_Y + 0x1000000
    assert f(0, Y, U, V, 10, 1, 3) == ss.SS_ERR_NULL
    assert f(X, Y, U, 0, 10, 1, 3) == ss.SS_ERR_NULL
    assert f(X, Y, U, V, 10, 1, 0) == ss.SS_ERR_BAD_SIZE
    assert f(X, Y, U, V, 10, 1, 3, 0) == ss.SS_ERR_BAD_SIZE
    assert f(X, Y, U, V, 10, 0, 3) == ss.SS_ERR_BAD_SIZE
    assert f(X, Y, U, V, 10, 1, 11) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert f(X, Y, U, V, 10 ** 6, 1, ss.SS_AFFINE_W_MAX + 1) == ss.SS_ERR_UNSUPPORTED
    assert f(X, Y, U, X + 4, 10, 1, 3) == ss.SS_ERR_OVERLAP
    assert f(X, Y, V + 8, V, 10, 1, 3) == ss.SS_ERR_OVERLAP
    assert f(X, Y, U, V + 2, 10, 1, 3) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_launch_count() == 0


def test_backward_validation(ss):
    # every invalid call returns its status before any launch (no GPU needed)
    X, G, D = FAKE_X, FAKE_X + 0x1000000, FAKE_Y
    assert ss.ss_pool_sum_backward(0, D, 10, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_NULL
    assert ss.ss_pool_sum_backward(G, D, 10, 1, 0, 1, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_sum_backward(G, D, 10, 1, 3, 0, ss.SS_F32) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_pool_sum_backward(G, D, 2, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_pool_sum_backward(G, G + 4, 10, 1, 3, 1, ss.SS_F32) == ss.SS_ERR_OVERLAP
    assert ss.ss_pool_sum_backward(G, D, 10, 1, 3, 1, 7) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_pool_max_backward(X, G, D, 10, 1, 3, 1, ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_pool_max_backward(0, G, D, 10, 1, 3, 1) == ss.SS_ERR_NULL
    assert ss.ss_pool_max_backward(X, G, X + 8, 10, 1, 3, 1) == ss.SS_ERR_OVERLAP
    assert ss.ss_conv1d_backward_input(G, D, 10, 1, None, 3, 1) == ss.SS_ERR_NULL
    assert ss.ss_conv1d_backward_input(G, D, 10, 1, [1.0] * 3, 3, 1, ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_conv1d_backward_input(G, D, 2000, 1, [1.0] * 1025, 1025, 1) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_conv1d_backward_filter_workspace(0) == 0
    assert ss.ss_conv1d_backward_filter_workspace(63) > 0
    assert ss.ss_conv1d_backward_filter(X, G, D, 10, 1, 3, 1, 0, 0) == ss.SS_ERR_BAD_SIZE  # no workspace
    assert ss.ss_conv1d_backward_filter(X, G, D, 10, 1, 11, 1, D + 4096, 1 << 20) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_pool2d_backward(0, G, D, 1, 8, 8, 2, 2, 2, 2, ss.SS_POOL_MAX) == ss.SS_ERR_NULL
    assert ss.ss_pool2d_backward(X, G, D, 1, 8, 8, 9, 2, 2, 2, ss.SS_POOL_AVG) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_pool2d_backward(X, G, D, 1, 8, 8, 2, 2, 2, 2, 5) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_launch_count() == 0


def test_conv2d_validation(ss):
    X, Y = FAKE_X, FAKE_Y
    f = [1.0] * 9
    assert ss.ss_conv2d(0, Y, 1, 8, 8, f, 3, 3) == ss.SS_ERR_NULL
    assert ss.ss_conv2d(X, Y, 1, 8, 8, None, 3, 3) == ss.SS_ERR_NULL
    assert ss.ss_conv2d(X, Y, 0, 8, 8, f, 3, 3) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv2d(X, Y, 1, 8, 8, f, 3, 3, 0, 1) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv2d(X, Y, 1, 2, 8, f, 3, 3) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv2d(X, Y, 1, 8, 8, f, 3, 3, 1, 1, ss.SS_I32) == ss.SS_ERR_UNSUPPORTED
    assert ss.ss_conv2d(X, X + 16, 1, 8, 8, f, 3, 3) == ss.SS_ERR_OVERLAP
    assert ss.ss_conv2d(X + 2, Y, 1, 8, 8, f, 3, 3) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_launch_count() == 0


def test_conv1d_mc_validation(ss):
    X, W, Y = FAKE_X, FAKE_X + 0x1000000, FAKE_Y
    assert ss.ss_conv1d_mc(0, W, Y, 1, 100, 64, 64, 3) == ss.SS_ERR_NULL
    assert ss.ss_conv1d_mc(X, W, Y, 0, 100, 64, 64, 3) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv1d_mc(X, W, Y, 1, 100, 64, 64, 0) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv1d_mc(X, W, Y, 1, 2, 64, 64, 3) == ss.SS_ERR_WINDOW_EXCEEDS_INPUT
    assert ss.ss_conv1d_mc(X + 1, W, Y, 1, 100, 64, 64, 3) == ss.SS_ERR_BAD_SIZE
    assert ss.ss_conv1d_mc(X, W, X + 64, 1, 100, 64, 64, 3) == ss.SS_ERR_OVERLAP
    assert ss.ss_launch_count() == 0


def test_missing_library_fails_loudly(tmp_path):
    # the product path has no CPU fallback: a package without libss.so refuses to import
    import shutil
    import sys
    pkg = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2305_16513_b200")
    dst = tmp_path / "paper_2305_16513_b200"
    shutil.copytree(pkg, dst, ignore=shutil.ignore_patterns("*.so", "csrc", "__pycache__"))
    r = subprocess.run([sys.executable, "-c", "import paper_2305_16513_b200"], cwd=tmp_path, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode != 0 and "ImportError" in r.stderr
