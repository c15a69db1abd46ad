"""CPU: the drop-in's grf::Xoshiro256Stream reproduces the reference's seeded
stream bit for bit (random.cpp:56-108): normals and raw xoshiro256++ words
against tests/golden/xoshiro_streams.npz (made from the reference build by
tests/golden/make_stream_golden.py) and, where oracle/_ref exists, live."""
import os
import subprocess

import numpy as np
import pytest

from oracle import pyoracle as po

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DUMP = os.path.join(ROOT, "paper_1105_2737_b200", "build", "stream_dump")
GOLD = os.path.join(ROOT, "tests", "golden", "xoshiro_streams.npz")


def dropin(seed, sub, n):
    out = subprocess.run([DUMP, str(seed), str(sub), str(n)], check=True, capture_output=True, text=True).stdout.split()
    normals = np.array([float.fromhex(x) for x in out[:n]])
    words = np.array([int(x) for x in out[n:]], np.uint64)
    return normals, words


def test_dropin_stream_matches_reference_golden():
    g = np.load(GOLD)
    keys = sorted({k.split("_")[0] for k in g.files})
    assert len(keys) >= 4
    tails = 0
    for k in keys:
        seed, sub = (int(v) for v in g[k + "_key"])
        want_n, want_w = g[k + "_normals"], g[k + "_words"]
        got_n, got_w = dropin(seed, sub, len(want_n))
        assert np.array_equal(got_w[:len(want_w)], want_w), k
        assert np.array_equal(got_n, want_n), (k, int(np.argmax(got_n != want_n)))
        tails += int((np.abs(want_n) > 3.6541528853610088).sum())
    assert tails > 0  # the fixture exercises the ziggurat tail branch


@pytest.mark.skipif(not os.path.exists(po.REF_LIB), reason="oracle/_ref is built only where /root/reference exists")
def test_dropin_stream_matches_reference_live():
    ref = po.Reference()
    for seed, sub in ((7, 0), (123456789, 5), (2**40 + 3, 1)):
        want_n, want_w = ref.xoshiro(seed, sub, 3000)
        got_n, got_w = dropin(seed, sub, 3000)
        assert np.array_equal(got_w, want_w) and np.array_equal(got_n, want_n), (seed, sub)
