"""Accuracy of the int8-sliced tcgen05 fp64 GEMM (csrc/ozaki_gemm.cuh) against
a long-double product, through tools/ozaki_test.cu built with nvcc for sm_100a.

Bound stated by the kernel: |ΔC| ≤ K·11·2⁻⁵⁶·s_a·s_b ≤ K·2^{-50.5}·max|a|·max|b|
(slicing remainders + dropped slice products; the int32 accumulation is exact).
Shapes: the c2 and c3 products (Y·W and Yᵀ⟨S⟩ with split-K partials), ragged
edges included (M, N, P not multiples of the 128-row tiles)."""
import os
import re
import subprocess

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

BOUND = 2.0 ** -50.5


@pytest.fixture(scope="module")
def tool(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("oz") / "ozaki_test")
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-I",
                    os.path.join(ROOT, "paper_1908_06843_b200", "csrc"), os.path.join(ROOT, "tools", "ozaki_test.cu"),
                    "-o", exe], check=True, timeout=600)
    return exe


@pytest.mark.parametrize("m,n,k,p", [(3001, 300, 256, 5003), (1500, 1000, 576, 2500), (777, 20, 100, 1000)])
def test_sliced_gemm_error_bound(tool, m, n, k, p):
    out = subprocess.run([tool, str(m), str(n), str(k), str(p)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    errs = [float(x) for x in re.findall(r"err/\([KP]·max\|a\|·max\|b\|\) = ([0-9.eE+-]+)", out.stdout)]
    rels = [float(x) for x in re.findall(r"err/Σ\|ab\| = ([0-9.eE+-]+)", out.stdout)]
    assert len(errs) == 2 and len(rels) == 2, out.stdout
    assert max(errs) <= BOUND, out.stdout
    assert max(rels) < 1e-14, out.stdout
