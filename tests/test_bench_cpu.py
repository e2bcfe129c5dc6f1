"""CPU legs of bench.py (no GPU): the reference arm's sampled CPU baseline for
configs too large for the reference (cfg5a), and the batch arm's sample
(cfg5b). These are the numbers the bench line reports beside the GPU ones, so
their scaling arithmetic is tested here at small sizes."""
import argparse
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _args(**kw):
    base = dict(gpus=1, steps=1, warmup=0, impl="reference", n=None, config="cfg2a",
                lu_mode="exact", no_cpu_baseline=False, no_e2e=False, count=4096)
    base.update(kw)
    return argparse.Namespace(**base)


def test_reference_sample_extrapolates_large_n(monkeypatch, orc):
    import bench
    from paper_2311_14616_b200 import configs
    monkeypatch.setattr(bench, "SAMPLE_N", 96)
    args = _args(config="cfg1", n=192)
    wl = {**configs.config("cfg1", 96), "n": 192}
    dt, info = bench.reference_solve(args, wl, None, None)
    sf, ss = info["split_s"]["factor"], info["split_s"]["solve"]
    if sf:  # the compiled reference reports its split; the restatement does not
        assert dt == pytest.approx(sf * 8.0 + ss * 4.0)
    assert info["reason"] == "SmallBackwardError"
    assert "extrapolated to N=192" in info["sample"] and "N=96" in info["sample"]


def test_reference_small_n_is_one_full_solve(orc):
    import bench
    from paper_2311_14616_b200 import configs
    args = _args(config="cfg2a", n=128)
    wl = configs.config("cfg2a", 128)
    a, b = bench.to_tw(wl["a"], wl["tw"]), bench.to_tw(wl["b"], wl["tw"])
    dt, info = bench.reference_solve(args, wl, a, b)
    assert dt > 0 and info["sample"].startswith("one full cfg2a solve")
    assert info["cores"] == 1


def test_batch_cpu_sample_scales_to_the_whole_batch(orc):
    import bench_batch
    args = _args(config="cfg5b", count=64)
    out = bench_batch.cpu_sample(args, 64, seconds=0.2)
    assert out["value"] > 0 and out["cores"] >= 1
    assert out["reasons"] == ["SmallBackwardError"]
    assert "of 64 (N=64)" in out["sample"]


def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "cfg1", "--n", "128", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "s" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] in (
        "reference", "port")


def test_bench_spawns_its_own_ranks_for_gpus_gt_1():
    """`python bench.py --gpus 2` outside torchrun re-executes itself under
    torch.distributed.run with two ranks on 127.0.0.1 (here the reference arm on
    gloo: rank 0 prints the line, rank 1 exits without work)."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "cfg1",
                          "--n", "192"], capture_output=True, text=True, timeout=300,
                         env={k: v for k, v in os.environ.items()
                              if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["n"] == 192 and line["value"] > 0
