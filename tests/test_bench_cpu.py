"""bench.py's contract on the CPU side: the reference arm prints one JSON line
with the driver's keys (it runs the C port of the reference on host cores, no
GPU), including under a simulated non-zero rank (silent)."""

import json
import os
import subprocess
import sys

from conftest import ROOT

REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config")


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                           "--steps", "1", "--warmup", "3", "--ref-budget", "0.3", *args],
                          capture_output=True, text=True, env=env, timeout=300)


def test_reference_arm_json_line():
    r = _run()
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "hist/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("1920x1080")


def test_reference_arm_other_ranks_are_silent():
    r = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--gpus", "2")
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def _bench(*args, env=None):
    e = dict(os.environ, **(env or {}))
    e.pop("WORLD_SIZE", None)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                          capture_output=True, text=True, env=e, timeout=300)


def test_gpus_flag_self_launches_ranks():
    """`bench.py --gpus 2` (no launcher) starts 2 ranks under torch.distributed.run;
    rank 0 reports n_gpus 2, the frame shards [0,32)/[32,64) and the step time as
    the max over ranks (dry run: the plumbing without device work)."""
    r = _bench("--gpus", "2", "--dry-run", "--steps", "3", "--warmup", "3")
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2
    assert d["shares"] == [[0, 32, 0, 32], [32, 64, 0, 32]]
    assert d["ms_per_step"] == max(d["rank_ms"]) and d["rank_ms"][1] > d["rank_ms"][0]
    assert d["config"]["parallelism"] == "frame-shard x2"


def test_gpus_flag_bin_shards():
    r = _bench("--gpus", "2", "--dry-run", "--workload", "4k128", "--steps", "3", "--warmup", "3")
    assert r.returncode == 0, r.stderr
    d = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])
    assert d["shares"] == [[0, 1, 0, 64], [0, 1, 64, 128]]


def test_gpus_flag_fails_loudly_without_devices():
    """More ranks than visible GPUs: a clear error and a non-zero exit, never a
    silent N=1 run."""
    r = _bench("--gpus", "2", "--steps", "3", "--warmup", "3")
    assert r.returncode != 0
    assert "CUDA device" in r.stderr


def test_world_size_must_match_gpus_flag():
    e = dict(os.environ, RANK="0", LOCAL_RANK="0", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4",
                        "--steps", "3", "--warmup", "3"], capture_output=True, text=True,
                       env=e, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE" in r.stderr


def test_reference_arm_reports_n_gpus():
    r = _bench("--impl", "reference", "--gpus", "2", "--workload", "512", "--steps", "1",
               "--warmup", "3", "--ref-budget", "0.3")
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert d["config"]["key"] == "512" and "host_cpu" in d["config"]


def test_share_of_is_single_process_only():
    """--share-of N emulates rank 0's share of an N-GPU run on one process;
    it is refused under a multi-rank launch and for the replica workload."""
    r = _bench("--share-of", "4", "--workload", "512", "--steps", "3", "--warmup", "3")
    assert r.returncode == 2 and "share-of" in r.stderr
    e = dict(os.environ, RANK="0", LOCAL_RANK="0", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                        "--share-of", "4", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, env=e, timeout=300)
    assert r.returncode == 2 and "share-of" in r.stderr


def test_csv_row_schema(tmp_path):
    """--csv appends the reference's CSV columns plus the roofline columns."""
    sys.path.insert(0, ROOT)
    import bench

    line = {"value": 100.0, "steps": 5, "n_gpus": 1, "parity": "output crc32 == reference golden",
            "hbm_frac_step": 0.5, "roofline": {"traffic": 2.0e8},
            "config": {"histograms_per_step": 1, "host_cpu": "cpu model (4 threads)"}}
    path = tmp_path / "b.csv"
    bench.write_csv(str(path), line, bench.WORKLOADS["512"])
    bench.write_csv(str(path), line, bench.WORKLOADS["512"])
    rows = path.read_text().splitlines()
    from paper_1711_01919_b200.harness import CSV_HEADER
    assert rows[0] == CSV_HEADER + "," + bench.CSV_EXTRA and len(rows) == 3
    cols = rows[1].split(",")
    assert cols[0] == "single_pass" and cols[1:4] == ["512", "512", "32"] and cols[10] == "53891c64"
    assert cols[11] == "1" and cols[15] == "200000000"
