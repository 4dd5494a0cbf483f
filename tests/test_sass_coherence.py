"""CPU: the fused / NVLink kernels never read shard bytes through the
non-coherent read-only path.

k_fused_flow / k_fused_oneshot read back shard bytes written earlier in the
same kernel; k_symm_flow / k_symm2_flow read shard bytes a PEER GPU wrote
over NVLink during the kernel, after a system-scope flag acquire.  Those
reads must be weak coherent loads (``ld.global.cg``), never ``ld.global.nc``
(SASS ``LDG.*.CONSTANT``): an .nc load is outside the PTX memory model for
data written while the kernel runs, and its line may be stale.  The only
.nc loads allowed in these kernels are the 256-bit reads of the bf16
partials, which no thread writes.  Checked on the built library's SASS
(cuobjdump cross-disassembles sm_100a without a GPU).
"""

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2411_09510_b200", "libmxb200.so")
KERNELS = ("k_fused_flow", "k_fused_oneshot", "k_symm_flow", "k_symm2_flow")


_CACHE = {}


def _sass():
    """SASS of just the fused / NVLink kernels (cuobjdump --function on
    their entry symbols: seconds, where a whole-library dump takes minutes)."""
    if "sass" in _CACHE:
        return _CACHE["sass"]
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe) or not os.path.exists(LIB):
        pytest.skip("cuobjdump or libmxb200.so missing")
    syms = subprocess.run([exe, "-symbols", LIB], capture_output=True, text=True,
                          check=True).stdout
    # every element format of the bf16-output, B = 32 instantiations (all
    # instantiations share the templated load path; ~0.4 s per function)
    names = sorted({ln.split()[-1] for ln in syms.splitlines()
                    if "STO_ENTRY" in ln and any(k in ln for k in KERNELS)
                    and "I13__nv_bfloat16" in ln and "Li32E" in ln})
    assert names, "no fused / NVLink kernel entry points in libmxb200.so"
    out = subprocess.run([exe, "-sass", "-fun", ",".join(names), LIB], capture_output=True,
                         text=True, check=True).stdout
    _CACHE["sass"] = out
    return out


def test_no_noncoherent_shard_reads():
    funcs = re.split(r"\n\s*Function : ", _sass())[1:]
    seen, bad = 0, []
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        if not any(k in name for k in KERNELS):
            continue
        seen += 1
        for op in re.findall(r"\b(LDG\.[A-Z0-9_.]*)", f):
            if "CONSTANT" in op and ".256" not in op:
                bad.append((name[:80], op))
    assert seen >= 20, f"only {seen} fused/NVLink kernels found in the SASS"
    assert not bad, bad[:10]


def test_shard_reads_are_l1_bypassing():
    """The FP4 read-back of k_fused_flow is a 128-bit ld.global.cg
    (LDG.E.128.STRONG.GPU or LDG.E.EF.128 -- never cached in L1)."""
    funcs = re.split(r"\n\s*Function : ", _sass())[1:]
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        if "k_fused_flow" in name and "Li32ELi1ELi4E" in name:  # B=32, E2M1, 4 bits
            lds = re.findall(r"\b(LDG\.[A-Z0-9_.]*)", f)
            assert any(".128" in op and "CONSTANT" not in op for op in lds), lds
            return
    pytest.fail("k_fused_flow<*, 32, E2M1, 4> not found")


PUSH_KERNELS = ("k_push_dqsum", "k_push2_requant", "k_push2_decode")


def test_push_kernels_no_noncoherent_reads():
    """The push consumers (k_push.cu) read only bytes written during the
    call -- peer shards pushed over NVLink by the GEMM epilogues, the
    requantised chunks -- and the residual, which may alias the output: no
    load in them may take the non-coherent path, whatever its width."""
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe) or not os.path.exists(LIB):
        pytest.skip("cuobjdump or libmxb200.so missing")
    syms = subprocess.run([exe, "-symbols", LIB], capture_output=True, text=True,
                          check=True).stdout
    names = sorted({ln.split()[-1] for ln in syms.splitlines()
                    if "STO_ENTRY" in ln and any(k in ln for k in PUSH_KERNELS)})
    assert len(names) >= 18, names
    sass = subprocess.run([exe, "-sass", "-fun", ",".join(names), LIB], capture_output=True,
                          text=True, check=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)[1:]
    assert len(funcs) == len(names)
    bad = [(f.split("\n", 1)[0].strip()[:80], op) for f in funcs
           for op in re.findall(r"\b(LDG\.[A-Z0-9_.]*)", f) if "CONSTANT" in op]
    assert not bad, bad[:10]
