"""CPU checks of the C-ABI library: it loads without a GPU, exports every
symbol include/tzc_b200.h declares, validates descriptors into the
reference's error taxonomy, and plans kernels deterministically."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2101_08458_b200 import _capi
from paper_2101_08458_b200 import device as D

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tzc_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"TZC_API\s+[\w\s\*]+?\b(tzc_b200_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert header_functions() == sorted(_capi.EXPORTS)


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _capi.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    syms = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = [f for f in header_functions() if f not in syms]
    assert not missing, missing
    # nothing else leaks from the shared object: the C ABI plus the tzc::
    # C++ host-library API (include/tzc/tzc.hpp); kernels/runtime stay hidden
    leaked = sorted(s for s in syms if not (s.startswith(("tzc_", "_ZN3tzc", "_ZNK3tzc"))))
    assert not leaked, leaked


def test_loads_without_gpu_and_reports_no_device():
    L = _capi.lib()
    assert L.tzc_b200_version().startswith(b"tzc-b200")
    if not os.path.exists("/dev/nvidia0"):
        assert L.tzc_b200_device_ok() == 0


def _conv(**kw):
    base = dict(n=2, hp=10, wp=10, c=64, k=64, r=3, s=3, stride=1)
    base.update(kw)
    d, _ = D.conv_desc((base["n"], base["hp"], base["wp"], base["c"]), (base["k"], base["r"], base["s"], base["c"]),
                       base["stride"])
    return d


@pytest.mark.parametrize("kw,addr,kind", [
    (dict(hp=2), 16, "ShapeError"),        # filter does not fit the pre-padded input
    (dict(), 8, "InjectError"),            # TMA operand not 16-byte aligned
    (dict(stride=0), 16, "ShapeError"),
])
def test_validation_errors_map_to_reference_kinds(kw, addr, kind):
    d = _conv(**kw) if kw.get("stride", 1) else _conv()
    if kw.get("stride", 1) == 0:
        d.stride = 0
    ep = _capi.Epilogue(kind=_capi.EP_I32, scale=1.0)
    buf = C.c_void_p(addr)  # never dereferenced: validation fails first
    rc = _capi.lib().tzc_b200_conv2d_i8(C.byref(d), buf, buf, None, buf, C.byref(ep), None)
    with pytest.raises(_capi.TzcError) as e:
        _capi.check(rc)
    assert e.value.kind == kind


def test_null_inputs_are_missing_input():
    d = _conv()
    ep = _capi.Epilogue(kind=_capi.EP_I32, scale=1.0)
    rc = _capi.lib().tzc_b200_conv2d_i8(C.byref(d), None, None, None, None, C.byref(ep), None)
    with pytest.raises(_capi.TzcError) as e:
        _capi.check(rc)
    assert e.value.kind == "MissingInput"


def test_profile_mismatch_is_type_error():
    d = _conv()
    ep = _capi.Epilogue(kind=_capi.EP_I32, scale=1.0)
    buf = C.c_void_p(16)
    rc = _capi.lib().tzc_b200_conv2d_f16(C.byref(d), buf, buf, None, buf, C.byref(ep), None)
    with pytest.raises(_capi.TzcError) as e:
        _capi.check(rc)
    assert e.value.kind == "TypeError"


@pytest.mark.parametrize("layer", ["c2_3x3_64", "c3_1x1_256_128", "c4_3x3_256", "c5_3x3_512", "c5_1x1_512_2048"])
def test_plans_for_resnet_layers(layer):
    from paper_2101_08458_b200.workloads import RESNET50_V15
    L = next(x for x in RESNET50_V15 if x.name == layer)
    d, _ = D.conv_desc((32, L.h, L.h, L.c), (L.k, L.r, L.r, L.c), L.stride)
    p = D.plan_conv(d)
    # bm = rows per work unit (shifted-window: 128 x MT tiles)
    assert p["bm"] in (128, 256, 512) and p["bn"] in (64, 128, 256) and L.k % p["bn"] == 0
    assert p["bk_bytes"] in (64, 128) and (L.c % p["bk_bytes"] == 0)
    # 0: tiled GEMM (1x1 s1), 1: TMA im2col, 2: shifted-window weight-stationary (3x3 s1, small weights)
    want = 0 if (L.r == 1 and L.stride == 1) else (2 if layer in ("c2_3x3_64",) else 1)
    assert p["a_mode"] == want
    assert 1 <= p["grid"] <= 148 and p["smem_bytes"] <= 227 * 1024
    assert p["splits"] >= 1 and (p["workspace_bytes"] > 0) == (p["splits"] > 1)


def test_plan_gemm_4096():
    d = _capi.GemmDesc(profile=0, m=4096, n=4096, k=4096, b_kn=0)
    d.out = D.nhwc_layout(4096)
    p = D.plan_gemm(d)
    assert (p["tiles_m"], p["tiles_n"], p["splits"]) == (32, 16, 1)


def test_plan_stem_space_to_depth():
    from paper_2101_08458_b200.workloads import RESNET50_V15
    L = RESNET50_V15[0]
    d, _ = D.conv_desc((256, L.h, L.h, L.c), (L.k, L.r, L.r, L.c), L.stride)
    p = D.plan_conv(d)
    assert p["a_mode"] == 3 and p["bk_bytes"] == 16 and p["bn"] == 64


def test_problem_options_validation_and_candidates():
    """Per-descriptor plan options (the tuner's install path) need no device:
    unknown names are rejected, known ones install and clear."""
    from paper_2101_08458_b200 import device as D
    from paper_2101_08458_b200._capi import TzcError
    cands = D.tune_candidates()
    assert cands[0] == "" and len(cands) == 20 and "bn=128" in cands
    D.set_conv_plan((2, 10, 10, 64), (64, 3, 3, 64), 1, spec="bn=128;pingpong_kb=0")
    D.set_conv_plan((2, 10, 10, 64), (64, 3, 3, 64), 1, spec="")
    with pytest.raises(TzcError, match="unknown option"):
        D.set_conv_plan((2, 10, 10, 64), (64, 3, 3, 64), 1, spec="warp_speed=9")
    D.clear_tuning()


def test_plan_cache_save_load_roundtrip(tmp_path):
    """The text plan cache: installed per-descriptor plans are written one line
    per descriptor, cleared, loaded back (validated first), and a malformed
    file is refused without installing anything."""
    from paper_2101_08458_b200 import device as D
    D.clear_tuning()
    D.set_conv_plan((32, 58, 58, 64), (64, 3, 3, 64), 1, spec="ws_mt=2;ws_epi_groups=2")
    D.set_conv_plan((32, 30, 30, 256), (256, 3, 3, 256), 1, spec="splits=2")
    path = tmp_path / "plans.txt"
    assert D.save_tuning(path) == 2
    text = path.read_text()
    assert "ws_mt=2;ws_epi_groups=2" in text and "conv u8i8 n=32 hp=58" in text
    D.clear_tuning()
    assert D.save_tuning(tmp_path / "empty.txt") == 0
    assert D.load_tuning(path) == 2
    assert D.save_tuning(tmp_path / "again.txt") == 2
    assert (tmp_path / "again.txt").read_text() == text
    bad = tmp_path / "bad.txt"
    bad.write_text(text + "cdeadbeef ws_mt=2\n")
    D.clear_tuning()
    with pytest.raises(Exception, match="bad descriptor key"):
        D.load_tuning(bad)
    assert D.save_tuning(tmp_path / "none.txt") == 0  # nothing installed from the bad file
    bad.write_text(text.replace("ws_mt=2", "ws_mt=3"))
    with pytest.raises(Exception, match="illegal value"):
        D.load_tuning(bad)
    D.clear_tuning()
