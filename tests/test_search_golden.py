"""CPU: pin the scheme-search evaluator's algorithm to the
reference.  The oracle restatement of one evaluation -- per-rank codec round
trip of the stored float32 partials, float64 rank-order sum, relative
Frobenius error (mx/tpsim.py:234-302, mx/search.py:230-248) -- must give the
reference's own evaluator values (tests/golden/search.json, produced by
make_golden_search.py running the real mxcomm) bit for bit."""

import json
import os

import numpy as np
import pytest

from oracle import mx_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "search.json")) as f:
        g = json.load(f)
    z = np.load(os.path.join(HERE, "golden", "search_partials.npz"))
    return g, {k: z[k] for k in z.files}


def oracle_eval(parts, spec):
    sch = O.scheme(spec)
    ref = np.zeros(parts[0].shape, np.float64)
    red = np.zeros_like(ref)
    for p in parts:
        flat = p.astype(np.float64).ravel()
        ss, es = O.compress(flat, sch)
        dec = O.decompress(ss, es, flat.size, sch, np.float64).reshape(p.shape)
        ref += p.astype(np.float64)
        red += dec
    err = red - ref
    en, rn = float(np.linalg.norm(err.ravel())), float(np.linalg.norm(ref.ravel()))
    return 0.0 if en == 0.0 else en / rn * 100.0, float(np.max(np.abs(err)))


def test_oracle_reproduces_reference_evaluator(golden):
    g, arrays = golden
    for ci, c in enumerate(g["configs"]):
        parts = [arrays[f"c{ci}_r{r}"] for r in range(c["degree"])]
        assert parts[0].shape == tuple(c["input_shape"][:-1]) + (c["weight_shape"][1],)
        for spec in g["schemes"]:
            v, mx = oracle_eval(parts, spec)
            assert v == float.fromhex(c["evaluator"][spec]), (ci, spec)
            assert mx == float.fromhex(c["reports"][spec]["max_abs_err"]), (ci, spec)


def test_search_module_surface():
    import paper_2411_09510_b200 as m
    from paper_2411_09510_b200 import search

    assert m.make_simulation_evaluator is search.make_simulation_evaluator
    for name in ("DeviceReductionEvaluator", "make_activation_evaluator",
                 "simulation_partials", "load_activation_dump"):
        assert hasattr(search, name)
    for name in ("serialize_device", "deserialize_device"):
        assert hasattr(m, name)


def test_simulation_partials_match_reference_inputs(golden):
    """simulation_partials regenerates the reference's seeded partials (up
    to the host BLAS' last bits)."""
    from paper_2411_09510_b200.search import simulation_partials

    g, arrays = golden
    for ci, c in enumerate(g["configs"]):
        parts, pad = simulation_partials(c["degree"], c["seed"], tuple(c["input_shape"]),
                                         tuple(c["weight_shape"]))
        assert pad == c["padding"]
        for r, p in enumerate(parts):
            np.testing.assert_allclose(p, arrays[f"c{ci}_r{r}"], rtol=1e-5, atol=1e-4)
