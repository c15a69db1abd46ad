#!/usr/bin/env python
"""A/B of plan-time environment variants in one process (GPU box).

  python tools/ab_env.py --config c2 "GRFC_CLUSTER=8" "GRFC_CLUSTER=8 GRFC_CSLOTS=2" ...

Each variant's env is applied before its Plan is created (the library reads its
GRFC_* switches at plan creation); the first variant listed is always the
default (no overrides). Prints ms per batch (CUDA events, median of --iters) and
whether every field is bit-identical to the default's output.
"""
from __future__ import annotations

import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1105_2737_b200 import grfc  # noqa: E402


def make_density(c):
    d, fam = len(c["counts"]), c["density"]
    return grfc.Density.gaussian_cov(d, fam[1]) if fam[0] == "gauss" else grfc.Density.matern(d, fam[1], fam[2])


def run(cfg, env, iters, alg):
    # the overrides stay set for the whole variant: some switches are read at plan
    # creation, others (ring geometry, schedule) at every launch
    saved = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        c = bench.CONFIGS[cfg]
        plan = grfc.Plan(c["counts"], tuple(1.0 for _ in c["counts"]), make_density(c), alg,
                         grfc.F32 if c["dtype"] == "f32" else grfc.F64, device=0)
        n = c["fields"]
        out = plan.generate_tensor(0, 0, n)
        for _ in range(3):
            plan.generate_tensor(0, 0, n, out=out)
        torch.cuda.synchronize()
        ts = []
        for _ in range(iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            plan.generate_tensor(0, 0, n, out=out)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts), out, plan.path
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=15)
    ap.add_argument("--alg", type=int, default=1)
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    c = bench.CONFIGS[a.config]
    pts = 1
    for x in c["counts"]:
        pts *= x
    pts *= c["fields"]
    ref_ms, ref, path = run(a.config, {}, a.iters, a.alg)
    print(f"default [{path}]: {ref_ms:.4f} ms  {pts / ref_ms / 1e6:.1f} Gpts/s", flush=True)
    for v in a.variants:
        env = dict(kv.split("=", 1) for kv in v.split())
        try:
            ms, out, path = run(a.config, env, a.iters, a.alg)
        except Exception as e:  # noqa: BLE001
            print(f"{v}: FAILED {e}", flush=True)
            continue
        same = bool(torch.equal(out, ref))
        diff = float((out.double() - ref.double()).abs().max()) if not same else 0.0
        print(f"{v} [{path}]: {ms:.4f} ms  {pts / ms / 1e6:.1f} Gpts/s  bit-identical={same} maxdiff={diff:.3e}",
              flush=True)


if __name__ == "__main__":
    main()
