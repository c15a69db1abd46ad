"""Generates tests/golden/xoshiro_streams.npz from the REFERENCE's own
Xoshiro256Stream (oracle/_ref: proj/core compiled unmodified). Run here, where
/root/reference exists; the fixture is committed.

    python tests/golden/make_stream_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import pyoracle as po  # noqa: E402

# (seed, substream): the acceptance suite's shape streams and the estimator's substreams
STREAMS = [(0, 0), (5150, 0), (20260800, 3), (2**64 - 1, 2**63)]
N = 16000  # normals per stream: every layer, the wedges and (p ~ 1e-4 per draw) the tail
NW = 256  # raw words per stream


def main():
    ref = po.Reference()
    out = {}
    for i, (seed, sub) in enumerate(STREAMS):
        normals, words = ref.xoshiro(seed, sub, N)
        out[f"s{i}_key"] = np.array([seed, sub], np.uint64)
        out[f"s{i}_normals"] = normals
        out[f"s{i}_words"] = words[:NW]
    np.savez_compressed(os.path.join(os.path.dirname(os.path.abspath(__file__)), "xoshiro_streams.npz"), **out)


if __name__ == "__main__":
    main()
