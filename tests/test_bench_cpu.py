"""bench.py pieces that run without a GPU: the reference arm's JSON line (the driver
runs `bench.py --impl reference` beside our arm) and the roofline formula of
SURVEY §8d that our arm's `roofline` object is computed with."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "C0",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("IPv6 lookups/sec")
    assert d["unit"] == "G lookups/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    assert d["config"]["workload"] == "C0"
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert "sample" in cb
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the reference arm never maps the product library, and its config is our arm's
    assert d["product_library_mapped"] == []
    assert cb["kind"] == "reference"
    sys.path.insert(0, str(ROOT))
    import bench
    from oracle.workload import Workloads
    info = Workloads().info("C0")
    assert d["config"] == bench.shared_config(info, 1001, info.n_queries, 1)


def test_reference_arm_other_ranks_exit_quietly():
    env = {"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1", "PATH": "/usr/bin:/bin"}
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--workload", "C0",
                        "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


@pytest.fixture(scope="module")
def bench_mod():
    sys.path.insert(0, str(ROOT))
    import bench
    return bench


def test_roofline_formula_c1(bench_mod, lpm):
    """C1 (depth 4): the bound is L2 with the leaf and level 3 charged to it (T = 3),
    as SURVEY §8d's table has it, for the measured peaks bench.py reports."""
    info = lpm.workload_info("C1")
    geom = lpm.build_tree(lpm.build_intervals(lpm.workload_fib(info.fib_kind)), 1).geometry
    rl = bench_mod.roofline(geom, 1, l2_gbs=20926.0, smem_gbs=36533.0, hbm_gbs=6547.8)
    assert rl["T"] == 3 and rl["bound"] == "l2"
    assert rl["bytes_per_query"] == {"hbm": 17, "smem": 384, "l2": 257}
    assert rl["lps"] == pytest.approx(20926.0e9 / 257)
    assert rl["terms_glps"]["hbm"] == pytest.approx(6547.8 / 17)


def test_roofline_formula_small_tree_in_smem(bench_mod, lpm):
    """C0 (depth 2): every split fits shared memory; the formula takes the best over T,
    which stages the two internal levels and charges the leaf to L2 (staging the
    leaves too would charge 384 B/query to shared memory), bound by shared memory."""
    info = lpm.workload_info("C0")
    geom = lpm.build_tree(lpm.build_intervals(lpm.workload_fib(info.fib_kind)), 1).geometry
    rl = bench_mod.roofline(geom, 1, l2_gbs=20926.0, smem_gbs=36533.0, hbm_gbs=6547.8)
    assert geom.depth == 2 and rl["T"] == 2 and rl["bound"] == "smem"
    assert rl["lps"] == pytest.approx(36533.0e9 / 256)
    full = [bench_mod.roofline(geom, 1, 20926.0, 36533.0, 6547.8, smem_cap=c)["lps"] for c in (0, 1 << 30)]
    assert full[0] == pytest.approx(20926.0e9 / (3 * 128 + 1)) and full[1] == rl["lps"]
