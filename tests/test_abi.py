"""The C-ABI library loads and exports every symbol include/spmesl.h declares; host-side
validation and penalty helpers (no device compute calls: these run without a GPU)."""
import ctypes
import json
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def S():
    from paper_2203_15031_b200 import build
    build.build()
    import paper_2203_15031_b200 as S
    S.load()
    return S


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "spmesl.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(spmesl_[a-z_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(S):
    from paper_2203_15031_b200 import _lib
    L = S.load()
    decl = declared_symbols()
    assert len(decl) >= 12
    for name in decl:
        assert hasattr(L, name), name
    assert set(decl) == set(_lib.EXPORTS)


def test_struct_sizes_match_header(S):
    from paper_2203_15031_b200 import _lib
    o = _lib.default_options()
    assert o.struct_size == ctypes.sizeof(_lib.Options)
    assert o.max_inner == 10000 and o.standardize == 1 and o.symmetrize == 1
    assert o.sigma_floor == 1e-8 and o.device == -1


def test_penalty_helpers_paper_values(S, oracle):
    g = json.load(open(os.path.join(GOLD, "penalty_levels.json")))
    n, p = g["n"], g["p"]
    tol = 0.5 * 10 ** -g["printed_decimals"]
    assert abs(S.lambda_ub(n, p) - g["lambda_ub"]) <= tol
    assert abs(S.lambda_univ(n, p) - g["lambda_univ"]) <= tol
    assert abs(S.solve_k(p) - g["k"]) <= tol
    assert abs(S.lambda_pb(n, p) - g["lambda_pb"]) <= tol
    for (n, p) in [(50, 20), (100, 500), (200, 1000), (400, 5000), (500, 20000)]:
        assert S.lambda_univ(n, p) == pytest.approx(oracle.lambda_univ(n, p), rel=1e-14)
        assert S.lambda_ub(n, p) == pytest.approx(oracle.lambda_ub(n, p), rel=1e-14)
        assert S.lambda_pb(n, p) == pytest.approx(oracle.lambda_pb(n, p), rel=1e-9)
    assert math.isnan(S.lambda_univ(10, 2))


def _call(S, X, n, p, lam=0.3, tol=1e-4, max_iter=100, **kw):
    from paper_2203_15031_b200 import _lib
    o = _lib.default_options(**kw)
    T = np.empty((max(p, 1), max(p, 1)))
    sg = np.empty(max(p, 1))
    it = np.empty(max(p, 1), np.int32)
    ptr = None if X is None else ctypes.c_void_p(X.ctypes.data)
    return S.load().spmesl_fit_ex(ptr, n, p, lam, tol, max_iter, ctypes.byref(o),
                                  ctypes.c_void_p(T.ctypes.data), ctypes.c_void_p(sg.ctypes.data),
                                  ctypes.c_void_p(it.ctypes.data), None, None, None)


def test_argument_validation_before_any_cuda_call(S):
    X = np.asfortranarray(np.random.default_rng(0).standard_normal((10, 5)))
    assert _call(S, None, 10, 5) == -1
    assert _call(S, X, 1, 5) == -1
    assert _call(S, X, 10, 1) == -1
    assert _call(S, X, 10, 5, lam=-0.1) == -1
    assert _call(S, X, 10, 5, lam=float("nan")) == -1
    assert _call(S, X, 10, 5, tol=0.0) == -1
    assert _call(S, X, 10, 5, max_iter=0) == -1
    assert _call(S, X, 10, 5, max_inner=0) == -1
    assert _call(S, X, 10, 5, tile_cols=12) == -1
    assert _call(S, X, 10, 5, mode=2) == -1
    assert b"mode" in S.load().spmesl_last_error()


def test_missing_library_fails_loudly(tmp_path, monkeypatch):
    from paper_2203_15031_b200 import _lib
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    monkeypatch.setattr(_lib, "_lib", None)
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _lib.load()


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2203_15031_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.lower().replace("oracle-free", ""), f


def test_ctypes_layouts_match_the_c_header(tmp_path):
    """The ctypes mirrors of spmesl_options / spmesl_stats have the C structs' size and field
    offsets (compiled from include/spmesl.h with the host compiler; no GPU needed)."""
    import shutil
    import subprocess
    from paper_2203_15031_b200 import _lib
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no host C compiler")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    fields = {"spmesl_options": [f for f, _ in _lib.Options._fields_],
              "spmesl_stats": [f for f, _ in _lib.Stats._fields_]}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "spmesl.h"', "int main(void) {"]
    for struct, names in fields.items():
        lines.append(f'printf("{struct} size %zu\\n", sizeof({struct}));')
        for f in names:
            lines.append(f'printf("{struct} {f} %zu\\n", offsetof({struct}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run([cc, "-I", os.path.join(root, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split("\n")
    got = {}
    for ln in out:
        if ln.strip():
            struct, key, val = ln.split()
            got[(struct, key)] = int(val)
    for struct, cls in (("spmesl_options", _lib.Options), ("spmesl_stats", _lib.Stats)):
        assert got[(struct, "size")] == ctypes.sizeof(cls), struct
        for f in fields[struct]:
            assert got[(struct, f)] == getattr(cls, f).offset, (struct, f)


def test_multi_device_options_validated_before_cuda():
    """options.num_devices outside 0..64 is an argument error raised before any CUDA call."""
    import numpy as np
    import paper_2203_15031_b200 as S
    X = np.random.default_rng(0).standard_normal((20, 10))
    with pytest.raises(S.SpmeslError) as e:
        S.fit(X, 0.3, num_devices=-1)
    assert e.value.code == -1
    with pytest.raises(S.SpmeslError) as e:
        S.fit(X, 0.3, num_devices=65)
    assert e.value.code == -1
    with pytest.raises(S.SpmeslError) as e:       # options.exchange outside 0..2
        S.fit(X, 0.3, num_devices=1, exchange=3)
    assert e.value.code == -1
