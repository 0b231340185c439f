"""The bench.py JSON contract, checked on the committed bench line
(profiles/r02f_bench.json, this round's GPU run) and on the argument
defaults (CPU only)."""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_recorded_bench_line_has_the_contract_keys():
    d = json.loads((ROOT / "profiles" / "r02b_bench.json").read_text())
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "cpu_baseline",
              "clocks", "gpu_launches"):
        assert k in d, k
    assert d["metric"].startswith("ax_helm") and d["unit"] == "GDOF/s" and d["higher_is_better"] is True
    assert d["warmup"] >= 3 and d["gpu_launches"] >= d["steps"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    assert c["kind"] in ("reference", "port") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["matches_device_result"] is True
    k = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(k)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(k["reasons"])


def test_recorded_bench_line_round2_blocks():
    """Round-2 keys: the same-config CPU arm with its parity gates, the C3
    sweep with a clock record per entry, and C4 / C5 strong-scaled blocks."""
    d = json.loads((ROOT / "profiles" / "r02b_bench.json").read_text())
    c = d["cpu_baseline"]
    assert c["same_config"] is True and c["gate"]["strict_bit_exact"] is True
    assert c["gate"]["fast_normwise"] <= 1e-12
    sweep = d["lx_sweep"]
    assert {(e["lx"], e["mode"]) for e in sweep} == {(lx, m) for lx in range(2, 17) for m in ("fast", "strict")}
    for e in sweep:
        assert e["kernel_ms"] > 0 and e["hbm_gbs"] > 0 and {"sm_mhz", "reasons"} <= set(e["clocks"])
        assert e["c3"] == (e["lx"] <= 12)
    for key in ("c4", "c5"):
        b = d[key]
        assert b["elements_total"] == 1 << 21 and b["scaling"] == "strong" and b["target_efficiency"] == 0.85
        assert all("parallel_efficiency" in t for t in b["transports"].values())


def test_bench_defaults_are_the_headline_configuration():
    sys.path.insert(0, str(ROOT))
    import bench

    assert bench.LX == 8 and bench.NEL == 1 << 18 and bench.BYTES_PER_POINT == 72
    assert bench.flops_model(8, 32768) == 1_912_602_624  # frozen (reference tests/test_oracle.py:245)


def test_self_launch_runs_n_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself under
    torch.distributed.run with 2 ranks (gloo here: no GPU); --dry-run stops
    after the rank plumbing and rank 0 reports n_gpus = 2."""
    import os
    import subprocess

    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"],
                         env=env, capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["dry_run"] and sorted(d["ranks"]) == [0, 1]
    assert d["launcher"] == "torch.distributed.run"


def test_reference_problem_is_the_references_own_inputs():
    """bench.reference_problem (chunk-parallel, PCG64 advanced per chunk)
    reproduces mdg.bench._problem bit for bit (reference bench.py:41-47)."""
    import numpy as np
    import pytest

    ref = Path("/root/reference/pkg/src")
    if not ref.exists():
        pytest.skip("reference sources not present")
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ref))
    import bench
    from mdg import bench as mbench

    for lx, nel in ((8, 700), (5, 333), (12, 9)):
        _, want = mbench._problem(lx, nel)
        got = bench.reference_problem(nel, lx, chunk=128)
        for k in bench.ABI:
            assert np.array_equal(got[k], want[k]), (lx, nel, k)
