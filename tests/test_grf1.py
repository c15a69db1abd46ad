"""GRF1 on-disk format (reference include/grf/field_io.hpp:10-14,
src/field_io.cpp:60-107): the device batch writer grfc_write_grf1 (GPU) and
the host helpers, checked bit for bit against the reference's own
write_grf1 / read_grf1 (oracle/_ref)."""
import os

import numpy as np
import pytest
import torch

from oracle import pyoracle as po
from paper_1105_2737_b200 import grfc

needs_ref = pytest.mark.skipif(not po.reference_available(), reason="oracle/_ref not built")


@needs_ref
def test_host_image_matches_reference_writer(tmp_path):
    ref = po.Reference()
    counts, lengths = (4, 6), (1.5, 2.0)
    vals = np.random.default_rng(1).standard_normal(counts)
    vals.flat[3] = -0.0
    ref.write_grf1(tmp_path / "r.grf1", counts, lengths, vals)
    assert (tmp_path / "r.grf1").read_bytes() == grfc.grf1_bytes(counts, lengths, vals)
    c, l, v = grfc.read_grf1(tmp_path / "r.grf1")
    assert c == counts and l == lengths and v.tobytes() == vals.tobytes()
    # header layout (test_field_io.cpp:57-68)
    b = grfc.grf1_bytes((2,), (1.0,), [0.5, -0.25])
    assert len(b) == 4 + 4 + 4 + 8 + 8 + 16 and b[:4] == b"GRF1" and b[4] == 1 and b[8] == 1 and b[12] == 2


@needs_ref
def test_corrupt_files_rejected_like_reference(tmp_path):
    """test_field_io.cpp:70-92: both readers reject the same corruptions."""
    ref = po.Reference()
    good = grfc.grf1_bytes((4,), (1.0,), [1.0, 2.0, 3.0, 4.0])
    bad_version = bytearray(good)
    bad_version[4] = 2
    for blob, msg in [(b"GRG1" + good[4:], "bad magic"), (bytes(bad_version), "unsupported version"),
                      (good[:-3], "truncated"), (good + b"x", "trailing")]:
        p = tmp_path / "c.grf1"
        p.write_bytes(blob)
        with pytest.raises(RuntimeError, match=msg):
            grfc.read_grf1(p)
        with pytest.raises(po.OracleError, match=msg):
            ref.read_grf1(p)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("dtype", [grfc.F32, grfc.F64])
def test_device_batch_writer_bit_exact(tmp_path, dtype):
    ref = po.Reference()
    counts, lengths = ((512, 256), (1.0, 2.0)) if dtype == grfc.F32 else ((48, 20), (2.0, 1.0))
    plan = grfc.Plan(counts, lengths, grfc.Density.matern(2, 1.5, 0.1), grfc.ONE_FFT_OVERWRITE, dtype)
    n, f0 = 70, 5  # several pipeline chunks at 512x256
    plan.write_grf1(9, f0, n, str(tmp_path / "f_{field}.grf1"))
    want = plan.generate_tensor(9, f0, n).double().cpu().numpy()
    for i in (0, 1, 33, n - 1):
        c, l, v = ref.read_grf1(tmp_path / f"f_{f0 + i}.grf1")
        assert c == counts and l == lengths
        assert v.tobytes() == want[i].tobytes()
    assert len(os.listdir(tmp_path)) == n


@pytest.mark.gpu
def test_device_writer_errors(tmp_path):
    plan = grfc.Plan((8, 8), (1.0, 1.0), grfc.Density.gaussian_cov(2, 0.1), grfc.ONE_FFT_OVERWRITE, grfc.F64)
    plan.write_grf1(1, 0, 1, str(tmp_path / "one.grf1"))  # single field: plain path
    c, _, v = grfc.read_grf1(tmp_path / "one.grf1")
    assert c == (8, 8) and v.tobytes() == plan.generate_tensor(1, 0, 1)[0].cpu().numpy().tobytes()
    with pytest.raises(ValueError, match="placeholder"):
        plan.write_grf1(1, 0, 2, str(tmp_path / "x.grf1"))
    with pytest.raises(RuntimeError, match="cannot open"):
        plan.write_grf1(1, 0, 1, "/nonexistent/dir/x.grf1")
    torch.cuda.synchronize()
