"""The pipeline drop-in: the reference's run_pipeline
(proj/src/pipeline.cpp:56-179) with its kernel loop (:99-137) swapped for
one batch call of the product -- oracle/pipeline_dropin.cpp, which links the
reference's own partitioning, IPU-simulator replay (run_devices fed the
product's per-unit cells, bsp.cpp:142-171) and write_results (io.cpp:258-298).
The whole results text, summary block included, must equal the reference's
byte for byte: the SHA-256 digests of SURVEY Appendix B (the README smoke
run) and of acceptance criterion 9 (proj/tests/acceptance.cpp:572-609), and
the reference's own run on further configurations with band failures,
several simulated devices and both scheduling policies."""
import ctypes as C
import hashlib
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN_SO = os.path.join(ROOT, "oracle", "_ref", "libxband_dropin.so")


class DropinConfig(C.Structure):
    _fields_ = [("pairs", C.c_int64), ("length", C.c_int64), ("p_match", C.c_double),
                ("k", C.c_int32), ("uniform_seed", C.c_int32), ("seed", C.c_uint64),
                ("x", C.c_int32), ("band", C.c_int32), ("tiles", C.c_int32),
                ("devices", C.c_int32), ("multicomparison", C.c_int32), ("work_steal", C.c_int32)]


def cfg(pairs, length, p_match, x, band=1024, k=17, uniform=False, seed=42, tiles=8, devices=1,
        multi=False, steal=True):
    return DropinConfig(pairs, length, p_match, k, int(uniform), seed, x, band, tiles, devices,
                        int(multi), int(steal))


# README.md:57 smoke run (8 pairs, L=2000, p=0.9, X=15,
# defaults otherwise) and acceptance criterion 9's configuration
README_SMOKE = cfg(8, 2000, 0.9, 15)
README_SHA = "c70b2d58908500b46bcc4bb07a9ae224ab3015e1d46a413928448d427e8111ed"
C9 = cfg(12, 400, 0.85, 12, band=64, uniform=True, tiles=3, devices=2, multi=True)
C9_SHA = "1f3d6084841fc5693f3c85598f0f8cb9eda923192482c62a6216d2aa84600407"

MORE = {
    "band_failures": cfg(40, 1500, 0.8, 25, band=24, uniform=True, seed=7, devices=3),
    "static_policy_multi": cfg(30, 900, 0.88, 10, band=48, uniform=True, seed=11, tiles=4,
                               devices=4, multi=True, steal=False),
    "long_pairs": cfg(6, 6000, 0.9, 20, band=256, seed=3, devices=2),
    "low_identity": cfg(50, 700, 0.6, 8, band=32, uniform=True, seed=5, tiles=2),
}


@pytest.fixture(scope="module")
def dropin():
    if not os.path.exists(DROPIN_SO):
        pytest.skip("oracle/_ref/libxband_dropin.so not built (needs /root/reference at build time)")
    lib = C.CDLL(DROPIN_SO)
    for f in (lib.dropin_reference, lib.dropin_product):
        f.restype = C.c_int64
        f.argtypes = [C.POINTER(DropinConfig), C.c_char_p, C.c_int64, C.POINTER(C.c_int)]
    return lib


def run(fn, c):
    code = C.c_int(-1)
    n = fn(C.byref(c), None, 0, C.byref(code))
    buf = C.create_string_buffer(int(n) + 1)
    fn(C.byref(c), buf, n, C.byref(code))
    return buf.raw[:n], code.value


def test_reference_digests_pinned(dropin):
    """The harness drives the reference exactly as Appendix B did (no GPU)."""
    text, code = run(dropin.dropin_reference, README_SMOKE)
    assert code == 0 and hashlib.sha256(text).hexdigest() == README_SHA
    assert text.split(b"\n")[1] == b"0\tL\t801\t991\t991\t25447\t18"
    text, code = run(dropin.dropin_reference, C9)
    assert code == 0 and len(text) == 769 and hashlib.sha256(text).hexdigest() == C9_SHA


@pytest.mark.gpu
@pytest.mark.parametrize("name,c,sha", [("readme_smoke", README_SMOKE, README_SHA),
                                        ("acceptance_c9", C9, C9_SHA)])
def test_product_results_text_digest(dropin, name, c, sha):
    text, code = run(dropin.dropin_product, c)
    assert code == 0
    assert hashlib.sha256(text).hexdigest() == sha, text.decode()[-400:]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(MORE))
def test_product_results_text_equals_reference(dropin, name):
    ref, rc = run(dropin.dropin_reference, MORE[name])
    got, gc = run(dropin.dropin_product, MORE[name])
    assert gc == rc
    assert got == ref
    if name == "band_failures":
        assert rc == 3 and b"# failed" in ref
