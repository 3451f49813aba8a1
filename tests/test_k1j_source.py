"""K1j's generated source (csrc/k1_jit.cpp) on the CPU: it is what NVRTC
compiles at family upload on the GPU box, so here it must compile for sm_100a
without spills, carry every function's constants as literals, and refuse
families outside the fq domain (those run K1 / K1x)."""
import ctypes as C
import os
import re
import shutil
import subprocess

import pytest

from paper_2501_01046_b200 import _lib, minhash


def _source(fam, H, L):
    lib = _lib.load()
    n = lib.nd_k1j_source(fam.functions, H, L, None, 0)
    assert n > 0
    buf = C.create_string_buffer(n + 1)
    assert lib.nd_k1j_source(fam.functions, H, L, buf, n + 1) == n
    return buf.value.decode()


@pytest.mark.parametrize("H,L", [(128, 5), (37, 3), (256, 16)])
def test_k1j_source_has_every_constant(H, L):
    fam = minhash.derive_family(5, H, L)
    src = _source(fam, H, L)
    assert "extern \"C\" __global__" in src and f"#define L {L}" in src
    # q of every function appears as a literal in a rol() call
    qs = {int(m, 16) for m in re.findall(r"rol\([^,]+, ci\d, co\d, cf\d, (0x[0-9a-f]+)u", src)}
    assert qs == {fam.functions[i].base for i in range(H)}
    assert src.count("case ") == (H + 15) // 16  # passes of 16 functions


def test_k1j_source_refuses_other_families():
    lib = _lib.load()
    f = (_lib.NdHashFn * 1)()
    f[0].modulus, f[0].base = 257, 3
    assert lib.nd_k1j_source(f, 1, 5, None, 0) == -1
    fam = minhash.derive_family(5, 8, 20)
    assert lib.nd_k1j_source(fam.functions, 8, 20, None, 0) == -1  # L > 16


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not installed")
def test_k1j_source_compiles_for_sm100a_without_spills(tmp_path):
    fam = minhash.derive_family(5, 128, 5)
    src = tmp_path / "k1j.cu"
    src.write_text(_source(fam, 128, 5))
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    r = subprocess.run([nvcc, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-Xptxas", "-v", str(src), "-o", str(tmp_path / "k1j.cubin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "0 bytes spill stores" in r.stderr
    regs = int(re.search(r"Used (\d+) registers", r.stderr).group(1))
    assert regs <= 80  # 6 CTAs of 128 threads per SM
