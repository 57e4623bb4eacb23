"""CPU: the C-ABI library loads and exports every symbol include/gwasgls_b200.h declares (no
compute calls without a GPU), and the ctypes binding covers all of them."""

import os
import re
import subprocess

from conftest import REPO

HEADER = os.path.join(REPO, "include", "gwasgls_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for must in ("gg_potrf_f64", "gg_trsm_lower_f64", "gg_gls_epilogue_f64", "gg_gls_block_f64",
                 "gg_widen_i8_f64", "gg_small_spd_solve_f64", "gg_gls_dots_f64"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_1304_2272_b200 import _capi

    lib = _capi.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b(gg_[a-z0-9_]+)\b", out))
    assert set(declared_symbols()) <= exported


def test_binding_covers_header():
    from paper_1304_2272_b200 import _capi

    assert set(declared_symbols()) == set(_capi.SIGNATURES)


def test_host_only_entry_points():
    from paper_1304_2272_b200 import _capi

    lib = _capi.load_library()
    assert lib.gg_version().decode().startswith("gwasgls_b200")
    assert lib.gg_pad(1) == 128 and lib.gg_pad(128) == 128 and lib.gg_pad(129) == 256
    assert lib.gg_potrf_workspace_bytes(10000) >= 8 * 10112 * 128
    # 7 int8 slices (balanced 8-bit digits) per operand row over the k range, plus the row exponents
    assert lib.gg_gemm_ozaki_workspace_bytes(1000, 500, 300, 0) >= 7 * 1500 * 304 + 4 * 1500
    assert lib.gg_gemm_ozaki_workspace_bytes(1000, 1000, 300, 1) < \
        lib.gg_gemm_ozaki_workspace_bytes(1000, 1000, 300, 0)
    assert lib.gg_trtri_workspace_bytes(10000) > 0
    # exact-int32 bound of the int8 path: 127 up to n = 132,104, then shrinking
    assert lib.gg_i8_value_bound(10000) == 127 and lib.gg_i8_value_bound(132104) == 127 and lib.gg_i8_value_bound(132105) == 126
    assert lib.gg_i8_value_bound(150000) == 2147483647 // (128 * 150000) == 111
    # 7 tile-packed slices (112 KB per 128 x 128 tile of the triangle) + 2 np metadata ints
    assert lib.gg_i8_slices() == 7
    assert lib.gg_inverse_slices_bytes(1000) == 36 * 7 * 128 * 128
    assert lib.gg_slice_meta_ints(1000) == 2 * 1024
    # argument validation happens before any device work
    rc = lib.gg_trsm_lower_f64(0, 1, None, 128, None, 128, None, 128, None)
    assert rc == _capi.GG_EARG
    assert b"null" in lib.gg_last_error() or b"bad size" in lib.gg_last_error()


def test_sm100a_code_in_library():
    from paper_1304_2272_b200 import _capi

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", _capi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "DMMA" in out, "FP64 tensor-core (DMMA) instructions missing from the GEMM"


def test_every_ctypes_call_matches_declared_arity():
    """A C-ABI call with an extra or missing argument passes garbage as the stream pointer; catch
    it statically for every call site in the package, bench and tools."""
    import ast

    from paper_1304_2272_b200 import _capi

    files = ["bench.py", "__graft_entry__.py"]
    for d in ("paper_1304_2272_b200", "tools", "tests"):
        files += [os.path.join(d, f) for f in os.listdir(os.path.join(REPO, d)) if f.endswith(".py")]
    bad = []
    for f in files:
        tree = ast.parse(open(os.path.join(REPO, f)).read())
        for node in ast.walk(tree):
            if (isinstance(node, ast.Call) and isinstance(node.func, ast.Attribute)
                    and node.func.attr in _capi.SIGNATURES):
                want = len(_capi.SIGNATURES[node.func.attr][1])
                if len(node.args) != want:
                    bad.append((f, node.lineno, node.func.attr, len(node.args), want))
    assert not bad, bad


def test_argument_validation_without_a_gpu():
    """Every compute entry point validates its arguments before touching the device: bad sizes,
    null pointers and bad leading dimensions return GG_EARG / GG_EDIM with a message (this runs
    on the CPU box; no kernel is launched)."""
    from paper_1304_2272_b200 import _capi

    lib = _capi.load_library()
    EARG, EDIM = _capi.GG_EARG, _capi.GG_EDIM
    V = None
    cases = [
        (lib.gg_potrf_f64, (0, V, 1, 0, V, V, 128, V, V, V), EARG),
        (lib.gg_trtri_lower_f64, (0, V, 128, V, 128, V, V), EARG),
        (lib.gg_trsm_lower_i8, (0, 1, V, V, V, 16, V, 128, V, V), EARG),
        (lib.gg_trsm_lower_i8_partials, (10, 1, V, V, V, 16, 3, V, V, V, V, 0, V, 0, V, V),
         EARG),
        (lib.gg_gls_reduce_solve_f64, (10, 1, 3, V, V, V, V, V, V, V), EARG),
        (lib.gg_gls_block_f64, (10, 3, 1, V, V, V, V, V, V, V, V, 0, V, 0, V, V, V, V, V), EARG),
        (lib.gg_slice_inverse_i8, (0, V, 128, V, V, V), EARG),
        (lib.gg_slice_packed_inverse_i8, (0, V, V, V, V), EARG),
        (lib.gg_row_exponents_blockcyclic, (10, 128, 1, 1, 0, 0, V, 128, V, V), EARG),
        (lib.gg_slice_blockcyclic_i8, (10, 128, 1, 1, 0, 0, V, 128, V, V, V), EARG),
        (lib.gg_slice_meta_i8, (10, V, V, V), EARG),
        (lib.gg_narrow_f64_i8, (0, 1, V, 1, V, 1, V, V), EARG),
        (lib.gg_small_spd_solve_f64, (1, 0, V, V, V, V, V, V), EARG),
        (lib.gg_gls_dots_f64, (10, 1, 25, V, 128, V, 128, V, V, V, V), EARG),
        # Ozaki GEMM: null A, then a workspace smaller than gg_gemm_ozaki_workspace_bytes
        (lib.gg_gemm_ozaki_f64, (64, 64, 64, V, 1, 64, V, 1, 64, V, 64, 1.0, 0.0, 0, V, 0, V),
         EARG),
        (lib.gg_gemm_ozaki_f64, (64, 64, 64, 16, 1, 64, 16, 1, 64, 16, 64, 1.0, 0.0, 0, 16, 1,
                                 V), EARG),
    ]
    for fn, args, want in cases:
        rc = fn(*args)
        assert rc in (want, EDIM), (fn.__name__, rc)
        assert lib.gg_last_error(), fn.__name__
