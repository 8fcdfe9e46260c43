"""CPU-side checks of the C-ABI library: it builds, loads, exports every symbol declared in
include/fmm_b200.h, reports the missing device instead of falling back, and its host-side
synthetic generator follows SURVEY.md §8d."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fmm_b200.h")
LIB = os.path.join(ROOT, "paper_1203_0889_b200", "lib", "libfmm_b200.so")


def declared_functions():
    text = open(HEADER).read()
    return re.findall(r"^(?:int|void|const char\*)\s+(fmm_\w+)\(", text, flags=re.M)


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_1203_0889_b200", "csrc"), "-j8", "-s"],
                       check=True)
    from paper_1203_0889_b200 import _capi
    return _capi.load()


def test_header_and_binding_agree():
    from paper_1203_0889_b200 import _capi
    assert sorted(declared_functions()) == sorted(_capi.SIGNATURES)


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 30
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", LIB], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}$", out, flags=re.M), n


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", LIB], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_no_device_is_an_error_not_a_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_1203_0889_b200 import _capi, fmm
    with pytest.raises(fmm.FMMError) as ei:
        fmm.Context(order=4)
    assert ei.value.status == _capi.ERR_NO_DEVICE
    with pytest.raises(fmm.FMMError) as ei:
        fmm.m2l(3, np.zeros(10), [1.0, 0, 0])
    assert ei.value.status == _capi.ERR_NO_DEVICE


def test_config_validation_mirrors_reference_messages(lib):
    from paper_1203_0889_b200 import _capi, fmm
    cases = [(dict(order=0), _capi.ERR_ORDER, "expansion order must be >= 1"),
             (dict(n_crit=0), _capi.ERR_NCRIT, "n_crit must be >= 1"),
             (dict(theta=1.0), _capi.ERR_THETA, "theta must be in (0,1)"),
             (dict(theta=0.0), _capi.ERR_THETA, "theta must be in (0,1)")]
    for kw, st, msg in cases:
        with pytest.raises(fmm.FMMError, match=re.escape(msg)) as ei:
            fmm.Context(**kw)
        assert ei.value.status == st


def test_generator_configs(lib):
    from paper_1203_0889_b200 import fmm
    n = 4096
    c1 = fmm.generate_bodies(1, n, 1)
    assert np.array_equal(c1, fmm.generate_bodies(1, n, 1))
    assert np.abs(c1[:, :3]).max() <= 1.0 and (c1[:, 3] > 0).all() and (c1[:, 3] <= 1.0 / n).all()
    c3 = fmm.generate_bodies(3, n, 1)
    r = np.linalg.norm(c3[:, :3], axis=1)
    assert r.max() <= 100.0 and np.allclose(c3[:, 3], 1.0 / n)
    assert 0.5 < np.median(r) < 1.9  # Plummer half-mass radius ~1.305
    c5 = fmm.generate_bodies(5, n, 1)
    assert np.allclose(np.linalg.norm(c5[:, :3], axis=1), 1.0)
    assert np.abs(c5[:, 3]).max() <= 1.0 / n
    # position drawn before charge, z first (g++ right-to-left Vec3 arguments)
    import oracle
    orc = oracle.Oracle()
    lib_o = orc.lib
    lib_o.orc_rng_init.argtypes = [C.c_void_p, C.c_uint64]
    lib_o.orc_rng_uniform.restype = C.c_double
    lib_o.orc_rng_uniform.argtypes = [C.c_void_p, C.c_double, C.c_double]
    lib_o.orc_rng_uniform01.restype = C.c_double
    lib_o.orc_rng_uniform01.argtypes = [C.c_void_p]
    st = C.c_uint64()
    lib_o.orc_rng_init(C.byref(st), 1)
    z = lib_o.orc_rng_uniform(C.byref(st), -1.0, 1.0)
    y = lib_o.orc_rng_uniform(C.byref(st), -1.0, 1.0)
    x = lib_o.orc_rng_uniform(C.byref(st), -1.0, 1.0)
    q = (1.0 - lib_o.orc_rng_uniform01(C.byref(st))) / n
    assert np.array_equal(c1[0], [x, y, z, q])


def test_host_api_reference_shapes():
    from paper_1203_0889_b200 import fmm
    assert fmm.n_coef(6) == 56
    assert fmm.index_of(0, 0, 1) == 1 and fmm.index_of(1, 0, 0) == 3
    M = np.arange(20.0)
    f = fmm.m2p_flip(4, M)
    deg = fmm.exponents(3).sum(1)
    assert np.array_equal(f[deg % 2 == 0], M[deg % 2 == 0])
    assert np.array_equal(f[deg % 2 == 1], -M[deg % 2 == 1])
    assert np.array_equal(fmm.m2p_flip(4, f), M)
    cells = {"child_count": np.array([2, 0, 0]), "child_begin": np.array([1, 0, 0]),
             "radius": np.array([1.0, 0.5, 0.5])}
    assert fmm.split_pair(0, 1, cells) == [(1, 1), (2, 1)]
    assert fmm.split_pair(1, 0, cells) == [(1, 1), (1, 2)]
    assert fmm.split_pair(0, 0, cells) == [(1, 0), (2, 0)]
    with pytest.raises(fmm.FMMError, match="cannot split leaf pair"):
        fmm.split_pair(1, 2, cells)
