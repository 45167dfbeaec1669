"""The C-ABI library loads on a CPU-only host and exports every entry point that
include/mpc200.h declares; the Python binding wraps exactly those names.  No compute call
is made here (no GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "mpc200.h")
LIB = os.path.join(ROOT, "paper_2511_19711_b200", "libmpc200.so")


def declared():
    txt = open(HDR).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(mpc_[a-z0-9_]+)\s*\(", txt)))


def test_header_declares_the_boundary():
    names = declared()
    for n in ["mpc_share", "mpc_open", "mpc_mul", "mpc_trunc", "mpc_cmp", "mpc_exp", "mpc_recip",
              "mpc_softmax", "mpc_gelu", "mpc_relu", "mpc_max", "mpc_maxpool2d", "mpc_layernorm",
              "mpc_rsqrt", "mpc_silu", "mpc_sigmoid", "mpc_square"]:
        assert n in names, n


def test_library_exports_every_declared_symbol():
    if not os.path.exists(LIB):
        import importlib.util
        spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_2511_19711_b200", "build.py"))
        b = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(b)
        b.build()
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mpc_[a-z0-9_]+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(LIB)                       # loads without a GPU
    lib.mpc_version.restype = ctypes.c_char_p
    assert lib.mpc_version().startswith(b"mpc200")


def test_binding_wraps_the_declared_names():
    import paper_2511_19711_b200 as m
    assert set(m.EXPORTS) == set(declared())


def test_ctx_create_rejects_bad_config_without_gpu():
    # argument validation happens before any CUDA call
    import paper_2511_19711_b200.binding as b
    cfg = b.Config(0, 0, 15, 0, 1, 2, 3, None, None)          # frac_bits != 16
    h = b.VP()
    assert b._L.mpc_ctx_create(ctypes.byref(cfg), ctypes.byref(h)) == 2      # MPC_ERR_RANGE
    cfg = b.Config(7, 0, 16, 0, 1, 2, 3, None, None)          # unknown mode
    assert b._L.mpc_ctx_create(ctypes.byref(cfg), ctypes.byref(h)) == 1      # MPC_ERR_INVALID


def test_header_is_plain_c99():
    """The boundary header compiles as strict C99 (no C++ or torch types leak into it)."""
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Wextra", "-pedantic", "-Werror", "-fsyntax-only", "-x", "c", HDR],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
