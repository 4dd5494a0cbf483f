"""The NVLink kernel's multi-rank protocol on ONE device.

k_symm_flow does not care whether its peer pointers are remote: N "ranks"
are N concurrent launches on N streams of the same GPU, each with its own
symmetric-layout buffer, the peers' buffers passed as plain device
pointers.  Sizes are small enough that every rank's CTAs are co-resident
(the kernels spin on each other's flags).  This exercises the real
cross-rank flag publish/acquire, per-CTA epochs and slot double-buffering
over repeated calls at N = 2..8, bit-exact against the oracle and
identical on every rank (mx/netbench.py:415-419)."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import mx_oracle as O  # noqa: E402
from tests.golden import inputs  # noqa: E402


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2411_09510_b200 import _native

    return _native


def run_ranks(_native, spec, parts, calls, out_dtype=torch.float32, algo="oneshot",
              residuals=None):
    from paper_2411_09510_b200.formats import parse_scheme

    sch = parse_scheme(spec, extensions=True)
    cs = sch.to_c()
    sets = parts if isinstance(parts[0], list) else [parts]
    N, n = len(sets[0]), sets[0][0].numel()
    if algo == "oneshot":
        slot, flags_off, total, ctas = _native.symm_layout(n, cs, N)
    else:
        slot, _, flags_off, total, ctas = _native.symm_twoshot_layout(n, cs, N)
    bufs = [torch.zeros(total, dtype=torch.uint8, device="cuda") for _ in range(N)]
    bptr = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    fptr = torch.tensor([b.data_ptr() + flags_off for b in bufs], dtype=torch.int64, device="cuda")
    state = [torch.zeros(1 + ctas, dtype=torch.int32, device="cuda") for _ in range(N)]
    flag = [torch.empty(1, dtype=torch.int64, device="cuda") for _ in range(N)]
    lib = _native.load()
    for f in flag:
        lib.mx_nonfinite_reset(ctypes.c_void_p(f.data_ptr()), None)
    outs = [torch.empty(n, dtype=out_dtype, device="cuda") for _ in range(N)]
    streams = [torch.cuda.Stream() for _ in range(N)]

    def res(r):
        return ctypes.c_void_p(residuals[r].data_ptr()) if residuals is not None else None

    torch.cuda.synchronize()
    results = []
    for c in range(calls):
        xs = sets[c % len(sets)]
        # the rank streams are non-blocking: order each call after the
        # current stream's work (the previous call's result clones below)
        for st in streams:
            st.wait_stream(torch.cuda.current_stream())
        for r in range(N):
            st = streams[r]
            odt = _native.MX_F32 if out_dtype == torch.float32 else _native.MX_BF16
            common = (ctypes.c_void_p(state[r].data_ptr()), ctypes.c_void_p(state[r].data_ptr() + 4),
                      ctypes.c_void_p(flag[r].data_ptr()), ctypes.c_void_p(st.cuda_stream))
            if algo == "oneshot":
                rc = lib.mx_allreduce_symm(
                    ctypes.c_void_p(xs[r].data_ptr()), _native.MX_BF16, n, ctypes.byref(cs),
                    ctypes.c_void_p(bptr.data_ptr()), ctypes.c_void_p(fptr.data_ptr()), r, N,
                    slot, ctypes.c_void_p(outs[r].data_ptr()), odt, res(r), *common)
            else:
                rc = lib.mx_allreduce_symm_twoshot(
                    ctypes.c_void_p(xs[r].data_ptr()), _native.MX_BF16, n, ctypes.byref(cs),
                    ctypes.c_void_p(bptr.data_ptr()), ctypes.c_void_p(fptr.data_ptr()), r, N,
                    ctypes.c_void_p(outs[r].data_ptr()), odt, res(r), *common)
            _native.check(rc, "mx_allreduce_symm")
        torch.cuda.synchronize()
        assert all(int(s[0].item()) == 0 for s in state), "peer wait timed out"
        results.append([o.clone() for o in outs])
    torch.cuda.synchronize()
    return results


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp6_e3m2:16:e8m0", "int8:64:e8m0",
                                  "fp4_e2m1:16:e5m0", "fp5_e2m2:32:e5m0"])
def test_symm_multirank_bit_exact(lib, N, spec):
    n = 32 * 1024  # 4 CTAs per rank: all ranks co-resident
    sets = []
    x64s = []
    for it in range(3):
        x64 = [inputs.gauss_bf16(n, 4000 + 17 * it + r) for r in range(N)]
        x64s.append(x64)
        sets.append([torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64])
    # 5 calls cycle through 3 input sets: epochs 1..5, both slots, twice
    out = run_ranks(lib, spec, sets, 5)
    for c, outs in enumerate(out):
        ref = O.allreduce_oneshot(x64s[c % 3], O.scheme(spec))
        for r in range(N):
            assert np.array_equal(outs[r].cpu().numpy(), ref), (spec, N, c, r)


def test_symm_multirank_bf16_out(lib):
    N, n = 4, 16 * 1024
    x64 = [inputs.gauss_bf16(n, 77 + r) for r in range(N)]
    xs = [torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64]
    outs = run_ranks(lib, "fp4_e2m1:32:e8m0", xs, 3, out_dtype=torch.bfloat16)
    ref = torch.from_numpy(O.allreduce_oneshot(x64, O.scheme("fp4_e2m1:32:e8m0"))).to(torch.bfloat16)
    for call in outs:
        for o in call:
            assert torch.equal(o.cpu(), ref)


@pytest.mark.parametrize("N", [2, 3, 4, 8])
@pytest.mark.parametrize("spec", ["fp4_e2m1:32:e8m0", "fp6_e2m3:64:e8m0", "int8:16:e8m0",
                                  "fp4_e2m1:32:e5m0", "fp5_e2m2:64:e5m0"])
def test_symm_twoshot_multirank_bit_exact(lib, N, spec):
    """k_symm2_flow == the NCCL two-shot semantics (oracle allreduce_twoshot)."""
    n = N * 16 * 1024  # chunks of 16 units: 2 CTAs per rank
    sets, x64s = [], []
    for it in range(3):
        x64 = [inputs.gauss_bf16(n, 6000 + 31 * it + r) for r in range(N)]
        x64s.append(x64)
        sets.append([torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64])
    for out_dtype in (torch.float32, torch.bfloat16):
        out = run_ranks(lib, spec, sets, 5, out_dtype=out_dtype, algo="twoshot")
        for c, outs in enumerate(out):
            ref = torch.from_numpy(O.allreduce_twoshot(x64s[c % 3], O.scheme(spec))).to(out_dtype)
            for r in range(N):
                assert torch.equal(outs[r].cpu(), ref), (spec, N, c, r, out_dtype)


@pytest.mark.parametrize("algo", ["oneshot", "twoshot"])
@pytest.mark.parametrize("out_dtype", [torch.float32, torch.bfloat16])
def test_symm_multirank_residual_fused(lib, algo, out_dtype):
    """residual + all_reduce fused into K5 / K5b's store: every rank's output
    equals its own residual + the oracle sum, added in out_dtype (the
    unfused torch add) -- bit for bit."""
    N, n, spec = 4, 4 * 16 * 1024, "fp4_e2m1:32:e8m0"
    x64 = [inputs.gauss_bf16(n, 8100 + r) for r in range(N)]
    xs = [torch.from_numpy(x).to("cuda", torch.bfloat16) for x in x64]
    resid = [torch.from_numpy(inputs.gauss_bf16(n, 8200 + r)).to("cuda", out_dtype)
             for r in range(N)]
    outs = run_ranks(lib, spec, xs, 3, out_dtype=out_dtype, algo=algo, residuals=resid)
    f = O.allreduce_oneshot if algo == "oneshot" else O.allreduce_twoshot
    s = torch.from_numpy(f(x64, O.scheme(spec))).to(out_dtype)
    for call in outs:
        for r in range(N):
            assert torch.equal(call[r].cpu(), resid[r].cpu() + s), (algo, out_dtype, r)


def test_symm_capped_grid_unit_row_loop():
    """With the CTA cap forced to 3 (MXB200_SYMM_CTAS, read once per
    process) every CTA of K5 / K5b loops over several unit rows and the last
    rows are ragged; the randomised multi-rank sweep must stay bit-exact."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MXB200_SYMM_CTAS="3")
    r = subprocess.run([sys.executable, os.path.join(root, "scripts", "fuzz_symm.py"), "20", "5"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
