"""The C-ABI library loads and exports every symbol include/pa.h declares.
No GPU needed: only argument-validation paths that return before any device
work are exercised here."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pa.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pa_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module", autouse=True)
def lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "pa_build", os.path.join(ROOT, "paper_1805_02372_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    b.build()
    return ctypes.CDLL(b.LIB)


def test_header_declares_the_north_star_calls():
    names = _declared()
    for must in ("pa_create", "pa_hash", "pa_destroy", "pa_hash_batch"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_names_match_header():
    import paper_1805_02372_b200 as pa
    from paper_1805_02372_b200 import _lib
    assert sorted(_lib.EXPORTED) == _declared()
    for n in _declared():
        assert callable(getattr(pa, n)), n


def test_version_and_status_strings():
    import paper_1805_02372_b200 as pa
    assert pa.pa_version() == 100
    assert pa.pa_status_string(0) == "PA_OK"
    assert pa.pa_status_string(5) == "PA_ERR_PRECISION"


def test_struct_layouts_match_header():
    import paper_1805_02372_b200._lib as L
    assert ctypes.sizeof(L.pa_options) == 4 + 4 + 8 + 4 + 28
    assert ctypes.sizeof(L.pa_info) == 8 * 2 + 4 * 2 + 8 * 6
    o = L.pa_options_init()
    assert o.struct_size == ctypes.sizeof(L.pa_options) and o.route == 0


def test_invalid_lengths_rejected_before_device_work():
    import paper_1805_02372_b200 as pa
    for n, m in ((0, 1), (5, 0), (5, 6)):
        with pytest.raises(pa.PaError) as e:
            pa.pa_create(n, m, 0, 0)
        assert e.value.status == pa.PA_ERR_INVALID_ARG
        assert str(n) in pa.pa_last_error() and str(m) in pa.pa_last_error()


def test_null_handles_are_errors_not_crashes():
    import paper_1805_02372_b200 as pa
    with pytest.raises(pa.PaError):
        pa.pa_hash(0, 0, 0, 0)
    with pytest.raises(pa.PaError):
        pa.pa_get_info(0)
    pa.pa_destroy(0)  # safe on NULL


def test_bad_options_rejected():
    import paper_1805_02372_b200 as pa
    o = pa.pa_options_init()
    o.route = 7
    with pytest.raises(pa.PaError) as e:
        pa.pa_create_ex(10, 5, 0, o, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG


def test_planner_host_only():
    """pa_plan: route choice and transform length N >= n+m-1 (reading R4), even, smooth
    factors, without any device work."""
    import paper_1805_02372_b200 as pa
    import pa_synth as syn
    for name, cfg in syn.CONFIGS.items():
        n, m = cfg["n"], cfg["m"]
        p = pa.pa_plan(n, m)
        if p["route"] == pa.PA_ROUTE_BITPACKED:
            assert n * m <= 2 ** 26
            continue
        N = p["transform_len"]
        assert N >= n + m - 1 and N % 2 == 0, name
        assert p["n1"] * p["n2"] * 2 == N
        assert N <= 1.15 * (n + m - 1) + 64, (name, N / (n + m - 1))
        for f in (p["n1"], p["n2"]):
            for q in (2, 3, 5, 7):
                while f % q == 0:
                    f //= q
            assert f == 1
        assert p["n1"] % p["cols_per_cta"] == 0
    for n, m in ((1, 1), (2, 1), (65537, 3), (10 ** 9, 10 ** 6)):
        try:
            p = pa.pa_plan(n, m)
        except pa.PaError as e:
            assert e.status == pa.PA_ERR_UNSUPPORTED
            continue
        if p["route"] == pa.PA_ROUTE_TRANSFORM:
            assert p["transform_len"] >= n + m - 1
