"""K1j's generated source (csrc/k1_jit.cpp) on the CPU: it is what NVRTC
compiles at family upload on the GPU box, so here it must compile for sm_100a
without spills in its word loops, carry every function's constants as literals, and refuse
families outside the fq domain (those run K1 / K1x)."""
import ctypes as C
import os
import re
import shutil
import subprocess
import sys

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
    # q of every function appears as a literal in a rol() (fq) or rold() (dn) call
    qs = {int(m, 16) for m in re.findall(r"rold?\([^,]+, (?:ci|x\d_)\d, co\d, cf\d, (0x[0-9a-f]+)u",
                                         src)}
    assert qs == {fam.functions[i].base for i in range(H)}
    # passes of 32 functions (dn, the default; plus one for the rare function
    # dn cannot take)
    assert (H + 31) // 32 <= src.count("case ") <= (H + 31) // 32 + 1


def test_k1j_source_refuses_other_families():
    lib = _lib.load()
    f = (_lib.NdHashFn * 1)()
    f[0].modulus, f[0].base = 257, 3
    assert lib.nd_k1j_source(f, 1, 5, None, 0) == -1
    fam = minhash.derive_family(5, 8, 20)
    assert lib.nd_k1j_source(fam.functions, 8, 20, None, 0) == -1  # L > 16


def _loops(sass: str):
    """(instruction count, body) of every backward branch's loop"""
    ins = [(int(m.group(1), 16), m.group(2)) for m in
           re.finditer(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", sass)]
    out = []
    for a, t in ins:
        m = re.search(r"BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            tgt = int(m.group(1), 16)
            out.append([x for b, x in ins if tgt <= b <= a])
    return out


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not installed")
@pytest.mark.parametrize("arith", ["dn", "fq"])
def test_k1j_source_compiles_for_sm100a_without_loop_spills(tmp_path, arith):
    """registers within the CTAs per SM the shape asks for (dn: 32 functions
    per pass, 4 CTAs of 128 threads, <= 128 registers; fq: 16 functions, 6
    CTAs, <= 80) and no local-memory traffic inside the word loops (the
    outer per-32-item loop may spill a counter once per batch); dn's word
    loop is 7.8 SASS per HWE (999 per 4 windows x 32 functions)"""
    env = dict(os.environ, ND_K1J_ARITH=arith)
    code = ("import ctypes as C, sys; from paper_2501_01046_b200 import _lib, minhash; "
            "f = minhash.derive_family(5, 128, 5); lib = _lib.load(); "
            "n = lib.nd_k1j_source(f.functions, 128, 5, None, 0); "
            "b = C.create_string_buffer(n + 1); lib.nd_k1j_source(f.functions, 128, 5, b, n + 1); "
            "sys.stdout.write(b.value.decode())")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       cwd=root)
    assert r.returncode == 0, r.stderr
    src = tmp_path / "k1j.cu"
    src.write_text(r.stdout)
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    cubin = tmp_path / "k1j.cubin"
    r = subprocess.run([nvcc, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-Xptxas", "-v", str(src), "-o", str(cubin)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    regs = int(re.search(r"Used (\d+) registers", r.stderr).group(1))
    F, regs_max = (32, 128) if arith == "dn" else (16, 80)
    assert regs <= regs_max
    sass = subprocess.run([os.path.join(os.path.dirname(nvcc), "cuobjdump"), "-sass", str(cubin)],
                          capture_output=True, text=True, check=True).stdout
    hwe = 4 * F  # one word: 4 windows x F functions
    words = [b for b in _loops(sass) if 7 * hwe <= len(b) <= 9.5 * hwe]
    assert len(words) >= 128 // F
    for b in words:
        assert not any("LDL" in x or "STL" in x for x in b)
    if arith == "dn":
        # no state conversion: one I2FP per window (the shared c_out), not per HWE
        assert all(sum(x.startswith("I2FP") for x in b) <= 4 for b in words)
        per_hwe = min(len(b) for b in words) / hwe
        assert per_hwe < 7.9, per_hwe  # fq: 572 / 64 = 8.94


@pytest.mark.skipif(shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"),
                    reason="nvcc not installed")
@pytest.mark.parametrize("L", [1, 5, 16])
def test_k1j_u16_source_compiles_without_spills(tmp_path, L):
    """K1j over 16-bit units (codepoint documents below U+10000): the fq
    arithmetic with c5 = 2^-3 passed at launch, two windows per word, 32
    functions per pass within 4 CTAs' registers (<= 128) and no local memory"""
    lib = _lib.load()
    fam = minhash.derive_family(5, 128, L, minhash.ShingleUnit.CODEPOINT)
    n = lib.nd_k1j_source_units(fam.functions, 128, L, 2, None, 0)
    assert n > 0 and lib.nd_k1j_source_units(fam.functions, 128, L, 3, None, 0) == -1
    buf = C.create_string_buffer(n + 1)
    lib.nd_k1j_source_units(fam.functions, 128, L, 2, buf, n + 1)
    src_text = buf.value.decode()
    assert "#define UW 2" in src_text and "rold(" not in src_text.split("extern")[1]
    src = tmp_path / "k1j16.cu"
    src.write_text(src_text)
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    r = subprocess.run([nvcc, "-cubin", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                        "-Xptxas", "-v", str(src), "-o", str(tmp_path / "k.cubin")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert int(re.search(r"Used (\d+) registers", r.stderr).group(1)) <= 128
    assert "0 bytes spill stores" in r.stderr
