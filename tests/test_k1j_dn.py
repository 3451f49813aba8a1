"""K1j's dn arithmetic (csrc/k1_jit.cpp: the state as a negative denormal, no
I2FP) checked on the CPU: the plan's constants, run through a host emulation
of the generated roll (tests/k1dn_emu.c, IEEE single precision with the
device instructions' rounding), give the exact residue
(q c + c_out QLn + c_in) mod p on every byte pair at the quotient boundaries
and on random states, and signatures equal to the C oracle's
(minhash.cpp:133-162).  The GPU tests (test_gpu_k1j.py) run the kernel
itself."""
import ctypes as C
import os
import shutil
import subprocess

import numpy as np
import pytest

from oracle_bind import Oracle
from paper_2501_01046_b200 import _lib, minhash

HERE = os.path.dirname(os.path.abspath(__file__))
u32p = C.POINTER(C.c_uint32)


@pytest.fixture(scope="module")
def emu(tmp_path_factory):
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    so = tmp_path_factory.mktemp("emu") / "libk1dn.so"
    subprocess.run([gcc, "-O2", "-shared", "-fPIC", "-frounding-math", "-fno-fast-math",
                    os.path.join(HERE, "k1dn_emu.c"), "-o", str(so), "-lm"], check=True)
    lib = C.CDLL(str(so))
    lib.dn_rol.restype = C.c_uint32
    lib.dn_rol.argtypes = [u32p, C.c_uint32, C.c_uint32, C.c_uint32]
    lib.dn_check_edges.restype = C.c_uint64
    lib.dn_check_edges.argtypes = [u32p]
    lib.dn_check_random.restype = C.c_uint64
    lib.dn_check_random.argtypes = [u32p, C.c_uint64, C.c_uint64]
    lib.dn_signatures.argtypes = [u32p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint8),
                                  C.POINTER(C.c_uint64), C.c_uint64, C.c_uint32, u32p]
    return lib


def plan(fam, H, L):
    lib = _lib.load()
    n = lib.nd_k1j_plan(fam.functions, H, L, None, 0)
    assert n == H
    out = np.zeros((H, 12), np.uint32)
    assert lib.nd_k1j_plan(fam.functions, H, L, out.ctypes.data_as(u32p), H) == H
    return out


def dn_rows(rows):
    return np.ascontiguousarray(rows[rows[:, 2] > 0])


def row_ptr(rows, i):
    return rows[i].ctypes.data_as(u32p)


@pytest.mark.parametrize("seed,H,L", [(5, 128, 5), (5, 256, 5), (11, 64, 3), (7, 40, 16)])
def test_dn_plan_shape(seed, H, L):
    allrows = plan(minhash.derive_family(seed, H, L), H, L)
    assert sorted(allrows[:, 4].tolist()) == list(range(H))  # every function once
    rows = allrows[allrows[:, 2] > 0]  # g = 0: the rare fq functions
    assert len(rows) >= H * 0.9
    for P in np.unique(allrows[:, 0]):
        assert (allrows[:, 0] == P).sum() <= 32  # F = 32 functions per pass (dn default)
    for P in np.unique(rows[:, 0]):
        sel = rows[rows[:, 0] == P]
        assert len(sel) <= 32
        assert len(np.unique(sel[:, 2])) == 1  # one offset g per pass
        assert len(np.unique(sel[:, 1])) <= 4  # at most 4 w classes
        assert all((w & 0xFF) == 0 for w in sel[:, 3])
        for c in np.unique(sel[:, 1]):
            assert len(np.unique(sel[sel[:, 1] == c][:, 3])) == 1
    assert allrows[:, 0].max() + 1 <= (H + 15) // 16 + 2
    fam = minhash.derive_family(seed, H, L)
    for r in rows:
        f = fam.functions[int(r[4])]
        assert r[8] == f.modulus and r[5] == f.base
        assert r[7] in (f.modulus, (1 << 32) - f.modulus)
        e = (int(r[11]) >> 23) & 0xFF
        assert 30 <= e <= 254


@pytest.mark.parametrize("seed,H,L", [(5, 128, 5), (3, 64, 7)])
def test_dn_roll_exact_at_quotient_boundaries(emu, seed, H, L):
    rows = dn_rows(plan(minhash.derive_family(seed, H, L), H, L))
    for i in range(len(rows)):
        assert emu.dn_check_edges(row_ptr(rows, i)) == 0, rows[i]
        assert emu.dn_check_random(row_ptr(rows, i), 20000, 17 + i) == 0, rows[i]


def test_dn_roll_exact_h256_random(emu):
    H = 256
    rows = dn_rows(plan(minhash.derive_family(5, H, 5), H, 5))
    for i in range(len(rows)):
        assert emu.dn_check_random(row_ptr(rows, i), 20000, 101 + i) == 0, rows[i]


@pytest.mark.parametrize("seed,H,L", [(5, 128, 5), (9, 48, 3), (5, 32, 16)])
def test_dn_signatures_equal_oracle(emu, seed, H, L):
    fam = minhash.derive_family(seed, H, L)
    rows = dn_rows(plan(fam, H, L))
    cols = rows[:, 4].astype(np.int64)
    rng = np.random.default_rng(seed)
    lens = rng.integers(L, 400, 24)
    lens[:4] = [L, L + 1, L + 2, L + 3]
    texts = [rng.integers(0, 256, int(n), dtype=np.uint8) for n in lens]
    texts[5][:] = 0
    texts[6][:] = 255
    offs = np.zeros(len(texts) + 1, np.uint64)
    offs[1:] = np.cumsum(lens)
    data = np.concatenate(texts)
    got = np.zeros((len(texts), H), np.uint32)
    emu.dn_signatures(rows.ctypes.data_as(u32p), len(rows), L, data.ctypes.data_as(C.POINTER(C.c_uint8)),
                      offs.ctypes.data_as(C.POINTER(C.c_uint64)), len(texts), H,
                      got.ctypes.data_as(u32p))
    o = Oracle()
    want = o.signatures(data, offs, o.derive_family(seed, H, L), L=L)
    assert np.array_equal(got[:, cols], want[:, cols])


def test_dn_plan_off_with_fq():
    env = dict(os.environ, ND_K1J_ARITH="fq")
    code = ("from paper_2501_01046_b200 import _lib, minhash; f = minhash.derive_family(5, 16, 5);"
            "print(_lib.load().nd_k1j_plan(f.functions, 16, 5, None, 0))")
    r = subprocess.run(["python", "-c", code], env=env, capture_output=True, text=True,
                       cwd=os.path.dirname(HERE))
    assert r.stdout.strip() == "-1", r.stderr
