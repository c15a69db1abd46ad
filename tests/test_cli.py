"""The grf CLI (paper_1105_2737_b200/cpp/tools/grf_cli.cpp) end to end — the
reference's tests/test_cli.cpp cases restated (line refs per test) against
our binary. Generation needs the device, so most cases are GPU tests; the
usage-error paths fail before any device work and run on CPU."""
import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT
from paper_1105_2737_b200 import grfc

BIN = os.path.join(ROOT, "paper_1105_2737_b200", "build", "grf")


def run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([BIN] + args.split(), capture_output=True, text=True, timeout=600, env=e)
    return r.returncode, r.stdout, r.stderr


def lines(text):
    return [l for l in text.splitlines() if l]


def test_usage_errors_cpu():
    """test_cli.cpp:82-86, 188-192: odd counts, unknown flags/subcommands, bad density."""
    rc, _, err = run("generate --points 5,4 --out /tmp/should_not_exist.grf1")
    assert rc == 1 and "even" in err
    assert run("generate --points 4,4 --out /tmp/x.grf1 --bogus 3")[0] == 1
    assert run("frobnicate")[0] == 1
    assert run("generate --points 4,4 --density nope:a=1 --out /tmp/x.grf1")[0] == 1
    rc, _, err = run("generate --points 8 --format pgm --out /tmp/should_not_exist.pgm")
    assert rc == 1 and "2-dimensional" in err
    assert run("cov --points 8 --density test1d --lengths 6.28 --samples 0")[0] == 1
    assert run("converge --levels 1..4 --samples 100")[0] == 1
    assert run("converge --levels 2..13 --samples 100")[0] == 1
    assert run("bench --points 8,8 --repeat 2")[0] == 1


@pytest.mark.gpu
def test_generate_deterministic_and_formats(tmp_path):
    """test_cli.cpp:67-79, 88-96."""
    flags = "generate --points 4,4 --lengths 1,1 --density poly:m=1,k=1,l=1,n=2 --seed 7 --out "
    assert run(flags + str(tmp_path / "a.grf1"))[0] == 0
    assert run(flags + str(tmp_path / "b.grf1"))[0] == 0
    a = (tmp_path / "a.grf1").read_bytes()
    assert a and a == (tmp_path / "b.grf1").read_bytes()
    assert run(f"generate --points 8,8 --format pgm --seed 1 --out {tmp_path / 'img.pgm'}")[0] == 0
    assert (tmp_path / "img.pgm").read_bytes()[:3] == b"P5\n"
    assert run(f"generate --points 4,6 --format csv --out {tmp_path / 'f.csv'}")[0] == 0
    assert (tmp_path / "f.csv").read_text().splitlines()[0] == "x1,x2,value"


@pytest.mark.gpu
def test_generate_batch_matches_device_fields(tmp_path):
    """B200 addition: --count N streams N GRF1 files; file f is field (seed, f)."""
    rc, _, _ = run(f"generate --points 64,32 --algorithm one-fft --seed 3 --count 5 --out {tmp_path}/g_{{field}}.grf1")
    assert rc == 0
    plan = grfc.Plan((64, 32), (1.0, 1.0), grfc.Density.poly(2, 1.0, 1, 1, 2), grfc.ONE_FFT_OVERWRITE, grfc.F64)
    want = plan.generate_tensor(3, 0, 5).cpu().numpy()
    for f in range(5):
        _, _, v = grfc.read_grf1(tmp_path / f"g_{f}.grf1")
        assert v.tobytes() == want[f].tobytes()


@pytest.mark.gpu
def test_cov_rows_oracles_and_determinism():
    """test_cli.cpp:98-133."""
    rc, out, _ = run("cov --points 16 --lengths 6.283185307179586 --density test1d --samples 500 "
                     "--oracle closed-form --seed 3")
    assert rc == 0
    ls = lines(out)
    assert len(ls) == 17 and ls[0] == "lag1,estimate,oracle,abs_diff"
    assert all(l.count(",") == 3 for l in ls[1:])
    rc, _, err = run("cov --points 16 --density poly:m=1,k=1,l=1,n=2 --samples 10 --oracle closed-form")
    assert rc == 1 and "test1d" in err
    flags = "cov --points 8 --lengths 6.283185307179586 --density test1d --samples 2000 --seed 5 --oracle discrete"
    a, b, c = run(flags), run(flags, {"GRF_THREADS": "1"}), run(flags, {"GRF_THREADS": "3"})
    assert a[0] == 0 and a[1] == b[1] == c[1]


@pytest.mark.gpu
def test_converge_report_and_gate():
    """test_cli.cpp:135-169."""
    rc, out, _ = run("converge --levels 2..4 --samples 2000 --seed 2")
    ls = lines(out)
    assert len(ls) >= 4 and ls[0] == "level,cells,max_error,mc_floor"
    assert ls[1].startswith("2,4,") and ls[3].startswith("4,16,")
    assert ls[-1].startswith("# fitted_slope=") and rc == 2
    rc, out, _ = run("converge --levels 2..2 --samples 100 --seed 2")
    assert "# warning" in out and rc == 2
    floor = lambda o: float(lines(o)[1].rsplit(",", 1)[1])  # noqa: E731
    assert floor(run("converge --levels 2..2 --samples 100")[1]) == pytest.approx(0.2)
    assert floor(run("converge --levels 2..2 --samples 400")[1]) == pytest.approx(0.1)


@pytest.mark.gpu
def test_bench_csv():
    """test_cli.cpp:171-187: header, draws column last (256 / 284 / 256 at 16x16)."""
    rc, out, err = run("bench --points 16,16 --repeat 5 --seed 1")
    ls = lines(out)
    assert len(ls) == 4 and ls[0] == "algorithm,points,P,repeat,median_seconds,draws"
    assert ls[1].startswith("two-fft,16x16,256,5,") and ls[1].endswith(",256")
    assert ls[2].startswith("one-fft,") and ls[2].endswith(",284")
    assert ls[3].endswith(",256")
    assert rc in (0, 2) and "Gpts/s" in err
    rc, out, _ = run("bench --points 256,256 --points 64,64,64 --repeat 5 --batch 8")
    assert rc in (0, 2) and len(lines(out)) == 7
