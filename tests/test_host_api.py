"""CPU tests of the host side: reference API surface, MXC1 container,
C-ABI library loading / symbol export, and loud failure without a GPU."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2411_09510_b200 as mx
from oracle import mx_oracle as O
from paper_2411_09510_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "mxb200.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(mx_\w+)\(", hdr, re.M))
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    lib = _native.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.mx_abi_version() == 1


def test_host_only_abi_calls():
    s = mx.parse_scheme("fp4_e2m1:32:e8m0")
    assert _native.stream_nbytes(2 * 128 * 8192, s.to_c()) == (65536, 1048576)
    assert _native.shard_layout(70, s.to_c()) == (0, 32, 96)
    bad = _native.MxScheme(0, 0, 1, 8, 32)  # FloatMicro without exponent bits
    rc = _native.load().mx_scheme_check(ctypes.byref(bad))
    assert rc == -5 and b"exponent" in _native.load().mx_last_error()
    with pytest.raises(mx.UnknownScheme):
        _native.check(rc, "check")


def test_registry_and_parse():
    assert list(mx.ELEMENT_FORMATS) == ["fp4_e2m1", "fp5_e2m2", "fp5_e3m1", "fp5_e1m3",
                                        "fp4_e1m2", "fp3_e1m1", "fp2_e1m0", "int3", "int4", "int5"]
    s = mx.parse_scheme("fp4_e2m1:32:e8m0")
    assert s.effective_bits == 4.25 and s.name == "fp4_e2m1:32:e8m0"
    for bad in ["fp4_e2m1:32", "nope:32:e8m0", "fp4_e2m1:x:e8m0", "fp4_e2m1:0:e8m0",
                "fp4_e2m1:32:e9m0", "fp6_e2m3:32:e8m0"]:
        with pytest.raises(mx.UnknownScheme):
            mx.parse_scheme(bad)
    assert mx.parse_scheme("fp6_e2m3:32:e8m0", extensions=True).element.name == "fp6_e2m3"
    # SPEC.md:468 effective-bits table (E5M0)
    got = [round(float(mx.parse_scheme(f"{e}:{b}:e5m0").effective_bits), 1)
           for e in ["fp3_e1m1", "fp4_e2m1", "fp5_e2m2"] for b in [8, 16, 32]]
    assert got == [3.6, 3.3, 3.2, 4.6, 4.3, 4.2, 5.6, 5.3, 5.2]


def test_grids_match_oracle_and_spec():
    assert mx.enumerate_grid(mx.ELEMENT_FORMATS["fp4_e2m1"]).values.tolist() == \
        [0, .5, 1, 1.5, 2, 3, 4, 6]
    assert mx.emax(mx.ELEMENT_FORMATS["fp5_e2m2"]) == 2 and mx.emax(mx.ELEMENT_FORMATS["int5"]) == 3
    for name, fmt in {**mx.ELEMENT_FORMATS, **mx.EXTENSION_FORMATS}.items():
        kind = "float" if fmt.kind is mx.FormatKind.FLOAT_MICRO else "int"
        assert np.array_equal(mx.enumerate_grid(fmt).values,
                              O.element_grid(kind, fmt.exponent_bits, fmt.mantissa_bits)), name
    # INTn == E1M(n-2) up to a power of two
    for n in (3, 4, 5):
        gi = mx.enumerate_grid(mx.ELEMENT_FORMATS[f"int{n}"]).values
        gf = mx.enumerate_grid(mx.ElementFormat(mx.FormatKind.FLOAT_MICRO, 1, n - 2)).values
        assert np.array_equal(gi / gi[-1], gf / gf[-1])


def test_element_format_validation():
    with pytest.raises(ValueError):
        mx.ElementFormat(mx.FormatKind.FLOAT_MICRO, 0, 3)
    with pytest.raises(ValueError):
        mx.ElementFormat(mx.FormatKind.FLOAT_MICRO, 5, 3)  # 9 bits
    with pytest.raises(ValueError):
        mx.ScaleFormat(3)


def test_container_roundtrip_and_errors():
    s = mx.parse_scheme("fp4_e2m1:32:e8m0")
    ss, es = O.compress(np.linspace(-3, 5, 70), O.scheme(s.name))
    ct = mx.CompressedTensor(s, (70,), ss, es)
    blob = mx.serialize(ct)
    assert len(blob) == mx.serialized_nbytes(s, (70,)) == 28 + 3 + 35
    assert mx.deserialize(blob) == ct
    with pytest.raises(mx.BadMagic):
        mx.deserialize(b"XXC1" + blob[4:])
    with pytest.raises(mx.UnsupportedVersion):
        mx.deserialize(blob[:4] + b"\x02" + blob[5:])
    with pytest.raises(mx.TruncatedStream):
        mx.deserialize(blob[:-1])
    with pytest.raises(mx.MalformedHeader):
        mx.deserialize(blob + b"\x00")
    with pytest.raises(mx.TruncatedStream):
        mx.deserialize(blob[:10])
    assert mx.header_nbytes(3) == 44  # code, not SPEC.md:162's "24 + 3*4"
    ext = mx.parse_scheme("int8:32:e8m0", extensions=True)
    with pytest.raises(KeyError):  # like mx/codec.py:337-338
        mx.serialize(mx.CompressedTensor(ext, (1,), b"\x00", b"\x00"))


def test_block_error_bound():
    s = mx.parse_scheme("fp4_e2m1:32:e8m0")
    assert mx.block_error_bound(127, s) == 1.0 and mx.block_error_bound(0, s) == 0.0


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="CPU-only check")
def test_compute_fails_loudly_without_gpu():
    with pytest.raises(mx.NativeUnavailable):
        mx.compress_tensor(np.ones(64), mx.parse_scheme("fp4_e2m1:32:e8m0"))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2411_09510_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\"[\s\S]*?\"\"\"", "", src).replace(
                    "OracleBackend", ""), f
