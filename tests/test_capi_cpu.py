"""CPU: the C-ABI library loads, exports every symbol include/*.h declares, and
validates configs (reference error behaviour) without touching a GPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2502_12784_b200", "libvattn_b200.so")
HEADER = os.path.join(ROOT, "include", "vattn_b200.h")


def declared_functions(header=HEADER):
    src = open(header).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_]+\s*\*?\s*([a-z_0-9]+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2502_12784_b200", "csrc")], check=True)
    return C.CDLL(LIB)


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("mha_forward", "mha_backward", "mha_backward_workspace_bytes", "vattn_last_error",
              "mha_forward_host", "mha_backward_host", "mha_step_host"):
        assert f in fns, fns


TRAD_LIB = os.path.join(ROOT, "paper_2502_12784_b200", "libvattn_b200_traditional.so")
TRAD_HEADER = os.path.join(ROOT, "include", "vattn_b200_traditional.h")


@pytest.mark.parametrize("lib_path,header", [(LIB, HEADER), (TRAD_LIB, TRAD_HEADER)])
def test_library_exports_every_declared_symbol(lib, lib_path, header):
    nm = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (\w+)$", nm, flags=re.M))
    missing = [f for f in declared_functions(header) if f not in exported]
    assert declared_functions(header) and not missing, missing


def test_fused_library_does_not_link_cublas():
    """The hot path is hand-written; only the comparator library links cuBLAS."""
    ldd = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "cublas" not in ldd, ldd


def test_sm100a_code_only():
    """The library carries sm_100a SASS (tcgen05 / TMA), no PTX-JIT or other arch fallback."""
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out and "sm_90" not in out and "sm_80" not in out, out
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass or "UTCQMMA" in sass or "UTCMMA" in sass  # tcgen05.mma
    assert "UTMALDG" in sass  # TMA tile loads
    assert "LDTM" in sass and "STTM" in sass  # tcgen05.ld / tcgen05.st


class Cfg(C.Structure):
    _fields_ = [("batch", C.c_int32), ("heads", C.c_int32), ("seq_len", C.c_int32), ("head_dim", C.c_int32),
                ("causal", C.c_int32), ("softmax_scale", C.c_float), ("dtype", C.c_int32),
                ("dropout_p", C.c_float), ("seed", C.c_uint64), ("bh_offset", C.c_int32), ("bh_count", C.c_int32)]


def test_validation_matches_reference_errors(lib):
    lib.mha_forward.argtypes = [C.POINTER(Cfg)] + [C.c_void_p] * 6
    lib.vattn_last_error.restype = C.c_char_p
    lib.mha_backward_workspace_bytes.argtypes = [C.POINTER(Cfg)]
    lib.mha_backward_workspace_bytes.restype = C.c_size_t
    EINVAL, EUNSUP, ECUDA = 1, 3, 4
    bad = [Cfg(0, 1, 64, 64, 0, 0.0, 0), Cfg(1, 1, 0, 64, 0, 0.0, 0), Cfg(1, 1, 64, 64, 2, 0.0, 0),
           Cfg(1, 1, 64, 64, 0, 0.0, 7), Cfg(1, 1, 64, 64, 0, float("nan"), 0),
           Cfg(1, 1, 64, 64, 0, 0.0, 0, 1.0, 0), Cfg(1, 1, 64, 64, 0, 0.0, 0, -0.1, 0)]
    for c in bad:
        assert lib.mha_forward(C.byref(c), 16, 16, 16, 16, 16, None) == EINVAL
        assert lib.mha_backward_workspace_bytes(C.byref(c)) == 0
    lib.mha_forward(C.byref(bad[0]), 16, 16, 16, 16, 16, None)
    assert b"batch and heads must be positive" in lib.vattn_last_error()  # attention_forward.cpp:32
    assert lib.mha_forward(C.byref(Cfg(1, 1, 64, 96, 0, 0.0, 0)), 16, 16, 16, 16, 16, None) == EUNSUP
    ok = Cfg(1, 1, 64, 64, 0, 0.0, 0)
    assert lib.mha_forward(C.byref(ok), None, 16, 16, 16, 16, None) == EINVAL  # null pointer
    assert lib.mha_forward(C.byref(ok), 8, 16, 16, 16, 16, None) == EINVAL  # misaligned
    assert lib.mha_backward_workspace_bytes(C.byref(ok)) > 0
    # valid call on a host without an sm_100 device fails loudly -- never a CPU fallback
    rc = lib.mha_forward(C.byref(ok), 16, 16, 16, 16, 16, None)
    assert rc in (ECUDA,) or os.environ.get("CUDA_VISIBLE_DEVICES") not in (None, "")


def test_slab_validation(lib):
    """(b, h) slabs: [bh_offset, bh_offset + bh_count) must lie inside B*H."""
    lib.mha_backward_workspace_bytes.argtypes = [C.POINTER(Cfg)]
    lib.mha_backward_workspace_bytes.restype = C.c_size_t
    lib.mha_forward_host.argtypes = [C.POINTER(Cfg)] + [C.c_void_p] * 6
    whole = lib.mha_backward_workspace_bytes(C.byref(Cfg(2, 4, 256, 64, 0, 0.0, 0, 0.0, 0, 0, 0)))
    half = lib.mha_backward_workspace_bytes(C.byref(Cfg(2, 4, 256, 64, 0, 0.0, 0, 0.0, 0, 4, 4)))
    assert whole > 0 and 0 < half < whole
    for off, cnt in ((0, 9), (5, 4), (-1, 2), (3, 0), (0, -1)):
        assert lib.mha_backward_workspace_bytes(C.byref(Cfg(2, 4, 256, 64, 0, 0.0, 0, 0.0, 0, off, cnt))) == 0
        assert lib.mha_forward_host(C.byref(Cfg(2, 4, 256, 64, 0, 0.0, 0, 0.0, 0, off, cnt)),
                                    16, 16, 16, 16, 16, None) == 1  # EINVAL


def test_cpp_api_header_compiles():
    r = subprocess.run(["bash", "-c", f"echo '#include \"vattn_b200/mha.hpp\"' | g++ -std=c++17 -fsyntax-only "
                                      f"-I{ROOT}/include -I/usr/local/cuda/include -x c++ -"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_python_mirror_config_validation():
    # AttnConfig mirrors vattn::AttnConfig::validate / scale; importing the
    # package loads the .so but makes no device call.
    import paper_2502_12784_b200 as vb
    with pytest.raises(ValueError):
        vb.AttnConfig(seq_len=100, head_dim=64).validate()
    with pytest.raises(ValueError):
        vb.AttnConfig(seq_len=64, head_dim=64, dropout_p=1.0).validate()
    vb.AttnConfig(seq_len=100, head_dim=64).validate(strict_tiles=False)
    assert abs(vb.AttnConfig(seq_len=64, head_dim=64).scale() - 0.125) < 1e-9
    assert vb.lib.vattn_abi_version() == 4
