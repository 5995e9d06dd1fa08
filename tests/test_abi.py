"""The C-ABI library loads and exports every symbol include/pa.h declares.
No GPU needed: only argument-validation paths that return before any device
work are exercised here."""
import ctypes
import os
import re
import subprocess

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


def _c_layout(tmp_path, struct, fields):
    """sizeof / offsetof as the C compiler sees include/pa.h."""
    src = tmp_path / f"{struct}.c"
    body = "".join(f'    printf("%zu\\n", offsetof({struct}, {f}));\n' for f in fields)
    src.write_text(f'#include <stddef.h>\n#include <stdio.h>\n#include "pa.h"\nint main(void) {{\n'
                   f'    printf("%zu\\n", sizeof({struct}));\n{body}    return 0;\n}}\n')
    exe = tmp_path / f"{struct}.out"
    subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()
    return int(out[0]), [int(v) for v in out[1:]]


@pytest.mark.parametrize("struct", ["pa_options", "pa_info", "pa_kernel_time"])
def test_struct_layouts_match_header(tmp_path, struct):
    import paper_1805_02372_b200._lib as L
    cls = getattr(L, struct)
    names = [f for f, _ in cls._fields_]
    size, offs = _c_layout(tmp_path, struct, names)
    assert ctypes.sizeof(cls) == size
    assert [getattr(cls, f).offset for f in names] == offs
    if struct == "pa_options":
        o = L.pa_options_init()
        assert o.struct_size == size and o.route == 0 and o.batch_keys == 0 and o.max_transform_len == 0
        assert o.arith == 0 and o.device == -1


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
            # a column-split plan covers its longest block (<= ceil(n / blocks) + 127 bits) plus m
            nb = -(-n // p["column_blocks"]) if p["column_blocks"] > 1 else n
            assert p["transform_len"] >= min(n, nb) + m - 1


def test_workspace_size_is_host_only_and_adds_up():
    """pa_workspace_size needs no device: route (b) = reversed seed + staging; route (a) grows
    with batch_keys by whole per-key work buffers; the Eq. (4) split sums its blocks."""
    import paper_1805_02372_b200 as pa
    al = lambda b: (b + 255) // 256 * 256  # noqa: E731
    n, m = 4096, 1024
    stage = al((n + 31) // 32 * 4) + al((m + 31) // 32 * 4)
    assert pa.workspace_size(n, m, route="bitpacked") == al(((m + 31) // 32 + (n + 31) // 32 + 4) * 4) + stage
    n, m = 1_000_003, 250_000
    one = pa.workspace_size(n, m, route="transform")
    four = pa.workspace_size(n, m, route="transform", batch_keys=4)
    info = pa.pa_plan(n, m)
    assert one >= 32 * (info["transform_len"] // 2)
    assert four - one >= 3 * 16 * (info["transform_len"] // 2)
    split = pa.workspace_size(n, m, route="transform", max_transform_len=600_000)
    assert split >= 16 * (info["transform_len"] // 2)  # one spectrum per block, 16 B per complex point
    # an unsplit handle whose default plan already fits is unchanged by the cap
    assert pa.workspace_size(n, m, route="transform", max_transform_len=10**9) == one


def test_option_and_pointer_errors_before_device_work():
    import paper_1805_02372_b200 as pa
    with pytest.raises(pa.PaError) as e:
        pa.workspace_size(10_000, 5_000, route="transform", max_transform_len=5_000)
    assert e.value.status == pa.PA_ERR_UNSUPPORTED and "max_transform_len" in pa.pa_last_error()
    with pytest.raises(pa.PaError) as e:
        pa.workspace_size(100, 10, batch_keys=5000)
    assert e.value.status == pa.PA_ERR_INVALID_ARG and "batch_keys" in pa.pa_last_error()
    o = pa.make_options()
    o.plan_mode = 7
    with pytest.raises(pa.PaError) as e:
        pa.pa_workspace_size(100, 10, o)
    assert e.value.status == pa.PA_ERR_INVALID_ARG and "plan_mode" in pa.pa_last_error()
    # SURVEY 8(b) pa_options.arith: FP64 is the built arithmetic, the NTTs are refused by name
    for a, ok in ((pa.PA_ARITH_AUTO, True), (pa.PA_ARITH_FP64, True), (pa.PA_ARITH_NTT32, False),
                  (pa.PA_ARITH_NTT64, False), (9, False)):
        o = pa.make_options(route="transform")
        o.arith = a
        if ok:
            assert pa.pa_workspace_size(100_000, 10_000, o) > 0
        else:
            with pytest.raises(pa.PaError) as e:
                pa.pa_workspace_size(100_000, 10_000, o)
            assert "arith" in pa.pa_last_error()
    o = pa.make_options()
    o.device = -2
    with pytest.raises(pa.PaError) as e:
        pa.pa_workspace_size(100, 10, o)
    assert e.value.status == pa.PA_ERR_INVALID_ARG and "device" in pa.pa_last_error()
    with pytest.raises(pa.PaError) as e:
        pa.pa_create_ws(100, 10, 0, None, 0, 1 << 20, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG and "workspace" in pa.pa_last_error()
    with pytest.raises(pa.PaError) as e:
        pa.pa_seed_from_paper_eq1(0, 0, 10, 5, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG
    with pytest.raises(pa.PaError) as e:  # overlap is rejected from the pointer values alone
        pa.pa_seed_from_paper_eq1(1 << 20, (1 << 20) + 16, 1000, 100, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG and "overlap" in pa.pa_last_error()
    with pytest.raises(pa.PaError) as e:
        pa.pa_hash_fresh_batch(0, 0, 4, 0, 4, 0, 4, 1, 0)
    assert e.value.status == pa.PA_ERR_INVALID_ARG


def test_plan_splits_keys_beyond_one_transform():
    """pa_plan (host-only) reports the Eq. (4) column split pa_create falls back to when n + m
    exceeds what one transform plans, and no split below that."""
    import paper_1805_02372_b200 as pa
    assert pa.pa_plan(10**8, 2 * 10**7)["column_blocks"] == 1
    p = pa.pa_plan(10**9, 10**8)
    assert p["column_blocks"] > 1 and p["transform_len"] < 10**9 + 10**8
    p = pa.pa_plan(10**10, 10**7)
    assert p["column_blocks"] >= 28 and p["workspace_bytes"] < 180 * 2**30


def test_product_library_ignores_developer_overrides():
    """PA_* plan / variant overrides exist only in the PA_DEV build (libpa_dev.so): the product
    libpa.so plans the same with and without them; the developer build follows them."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\nimport paper_1805_02372_b200 as pa\n"
            "p = pa.pa_plan(10**7, 10**6); print(p['n1'], p['n2'], p['cols_per_cta'])\n" % ROOT)
    force = {"PA_FORCE_PLAN": "4096,3600,2", "PA_K13_ASC": "0", "PA_FORCE_T1": "100"}
    base = {k: v for k, v in os.environ.items() if k != "PA_LIB"}

    def plan(env):
        r = subprocess.run([sys.executable, "-c", code], env={**base, **env}, capture_output=True, text=True,
                           timeout=300, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        return r.stdout.strip()
    assert plan({}) == plan(force) != "4096 3600 2"
    dev = os.path.join(ROOT, "paper_1805_02372_b200", "libpa_dev.so")
    if os.path.exists(dev):
        assert plan({**force, "PA_LIB": dev}) == "4096 3600 2"
