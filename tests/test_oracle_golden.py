"""Pin the CPU oracle against vectors produced by the real reference.

Every GPU parity test compares against ``oracle/mx_oracle.py``; these tests
prove that oracle reproduces the reference (``tests/golden/make_golden.py``)
byte for byte before it is trusted.
"""

import hashlib

import numpy as np
import pytest

from oracle import mx_oracle as O
from tests.golden import inputs


def sha(b):
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def test_explicit_vectors(golden):
    assert len(golden["vectors"]) >= 10
    for v in golden["vectors"]:
        sch = O.scheme(v["scheme"])
        x = np.array([float.fromhex(h) for h in v["values_hex"]])
        ss, es = O.compress(x, sch)
        assert ss.hex() == v["scale_stream"], v["name"]
        assert es.hex() == v["element_stream"], v["name"]
        dec = O.decompress(ss, es, x.size, sch)
        assert [float(d).hex() for d in dec] == v["decoded_hex"], v["name"]


def test_spec_examples_literal():
    # SPEC.md:130  [1,-6,0.25,3] FP4/E8M0 -> stored 127, codes [2,15,0,5]
    st, codes = O.quantize(np.array([1.0, -6.0, 0.25, 3.0]), O.scheme("fp4_e2m1:32:e8m0"))
    assert st.tolist() == [127] and codes.tolist() == [2, 15, 0, 5]
    # SPEC.md:132  [2^130, 1] FP4/E5M0 -> stored 31, codes [7,0], decoded 393216
    sch = O.scheme("fp4_e2m1:32:e5m0")
    st, codes = O.quantize(np.array([2.0 ** 130, 1.0]), sch)
    assert st.tolist() == [31] and codes.tolist() == [7, 0]
    assert O.dequantize(st, codes, 2, sch).tolist() == [393216.0, 0.0]
    # signed zero keeps the sign bit in non-zero blocks
    st, codes = O.quantize(np.array([-0.1, 6, -0.0, 0]), O.scheme("fp4_e2m1:32:e8m0"))
    assert codes.tolist() == [8, 7, 8, 0]
    # FP4 grid
    assert O.element_grid("float", 2, 1).tolist() == [0, .5, 1, 1.5, 2, 3, 4, 6]


def test_wire_accounting_spec_148():
    sch = O.scheme("fp4_e2m1:32:e8m0")
    n = 2 * 128 * 8192
    ss, es = O.compress(np.zeros(n), sch)
    assert len(ss) == 65536 and len(es) == 1048576


@pytest.mark.parametrize("case", list(inputs.CASES))
def test_digest_sweep(golden, case):
    gen, _dtype = inputs.CASES[case]
    x = gen()
    g = golden["digests"][case]
    assert sha(x.astype(np.float64)) == g["input_sha"], "input generator drifted"
    bad = []
    for spec, d in g["schemes"].items():
        sch = O.scheme(spec)
        ss, es = O.compress(x, sch)
        if sha(ss) != d["scale"] or sha(es) != d["elem"]:
            bad.append(spec)
            continue
        if sha(O.decompress(ss, es, x.size, sch, np.float32)) != d["dec32"]:
            bad.append(spec + "/dec32")
        if sha(O.decompress(ss, es, x.size, sch, np.float64)) != d["dec64"]:
            bad.append(spec + "/dec64")
    assert not bad, bad


def test_decode_random_streams(golden):
    bad = []
    for spec, d in golden["decode"].items():
        sch = O.scheme(spec)
        n = d["n"]
        nb = -(-n // sch.block)
        ss, es = inputs.random_streams((nb * sch.kbits + 7) // 8, (n * sch.bits + 7) // 8, d["seed"])
        with np.errstate(over="ignore"):
            if sha(O.decompress(ss, es, n, sch, np.float32)) != d["dec32"]:
                bad.append(spec)
        if sha(O.decompress(ss, es, n, sch, np.float64)) != d["dec64"]:
            bad.append(spec + "/64")
    assert not bad, bad


def test_rank_order_reduction(golden):
    for spec, d in golden["reduce"].items():
        parts = [inputs.gauss_bf16(d["n"], s) for s in d["seeds"]]
        assert sha(O.allreduce_oneshot(parts, O.scheme(spec))) == d["sum32"], spec


def test_nonfinite(golden):
    for d in golden["nonfinite"]:
        x = np.ones(4099)
        x[d["index"]] = float(d["value"])
        x[4098] = np.nan
        assert O.first_nonfinite_block(x, d["block"]) == d["block_index"]


@pytest.mark.slow
def test_large_prefill_shape(golden):
    from paper_2411_09510_b200.synth import rank_partials
    g = golden["large"]
    p0, p1 = rank_partials(tuple(g["shape"]), 2, seed=0)
    assert [sha(p0), sha(p1)] == g["input_sha"]
    for spec in ["fp4_e2m1:32:e8m0", "fp6_e2m3:32:e8m0"]:
        sch = O.scheme(spec)
        ss, es = O.compress(p0, sch)
        assert sha(ss) == g[spec]["scale"] and sha(es) == g[spec]["elem"], spec
        assert sha(O.allreduce_oneshot([p0, p1], sch).reshape(g["shape"])) == g[spec]["tp2_sum32"]


def test_twoshot_chunks_block_aligned():
    for n, N, B in [(8388608, 8, 32), (4099, 3, 32), (100, 4, 7), (5, 8, 32)]:
        ch = O.twoshot_chunks(n, N, B)
        assert ch[0][0] == 0 and ch[-1][1] == n
        for lo, hi in ch[:-1]:
            assert (lo == n or lo % (8 * B) == 0) and (hi == n or hi % (8 * B) == 0)


def test_twoshot_equals_whole_tensor_codes_when_chunked():
    # per-chunk quantisation == whole-tensor quantisation
    sch = O.scheme("fp5_e2m2:32:e8m0")
    x = inputs.gauss_bf16(5000, 9)
    ss, es = O.compress(x, sch)
    st, codes = O.quantize(x, sch)
    parts_st, parts_codes = [], []
    for lo, hi in O.twoshot_chunks(x.size, 4, sch.block):
        a, b = O.quantize(x[lo:hi], sch)
        parts_st.append(a)
        parts_codes.append(b)
    assert np.array_equal(np.concatenate(parts_st), st)
    assert np.array_equal(np.concatenate(parts_codes), codes)
