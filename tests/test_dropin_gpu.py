"""GPU: the C++ grf:: drop-in (paper_1105_2737_b200/cpp) through its own test
program (the reference's test cases restated, tests/cpp/test_dropin.cpp) and
against the reference's golden fields via FixedStream injection."""
import os
import struct
import subprocess
import tempfile

import numpy as np
import pytest

from conftest import ROOT, golden_cases, rel_l2

pytestmark = pytest.mark.gpu

BIN = os.path.join(ROOT, "paper_1105_2737_b200", "build", "test_dropin")


def test_dropin_suite():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]


def test_dropin_stream_overload_matches_reference_golden(golden):
    n = 0
    with tempfile.TemporaryDirectory() as tmp:
        for key, counts, lengths, fam, rr, ii, alg, draws, field in golden_cases(golden):
            src, dst = os.path.join(tmp, "in.bin"), os.path.join(tmp, "out.bin")
            with open(src, "wb") as f:
                d = len(counts)
                f.write(struct.pack("<i", d))
                f.write(np.asarray(counts, np.int64).tobytes())
                f.write(np.asarray(lengths, np.float64).tobytes())
                f.write(struct.pack("<i", fam))
                f.write(np.asarray(rr, np.float64).tobytes())
                f.write(np.asarray(ii, np.int32).tobytes())
                f.write(struct.pack("<i", alg))
                f.write(struct.pack("<Q", len(draws)))
                f.write(np.asarray(draws, np.float64).tobytes())
            r = subprocess.run([BIN, "--synth", src, dst], capture_output=True, text=True, timeout=120)
            assert r.returncode == 0, (key, r.stderr)
            got = np.fromfile(dst, np.float64)
            assert rel_l2(got, field) <= 1e-12, (key, rel_l2(got, field))
            n += 1
    assert n >= 30
