"""Drop-in check in the reference's own C++ types: oracle/_ref/facade_demo runs
the reference's signature_batch / band_bucket_ids / compare_pass /
union_pairs+components and include/neardup_b200.hpp's neardup::b200
equivalents on the same corpus and exits non-zero on any difference."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_facade_matches_reference_in_its_own_types():
    exe = os.path.join(ROOT, "oracle", "_ref", "facade_demo")
    assert os.path.exists(exe), "build with `make -C oracle` (needs the reference sources)"
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FACADE OK" in r.stdout
