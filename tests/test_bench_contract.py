"""bench.py's reference arm (the CPU oracle, this tier's reference) keeps the driver's
JSON-line contract; under torchrun only rank 0 prints.  CPU only (c1 is tiny)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, gpus=1, drop_world=False):
    env = dict(os.environ, **(extra_env or {}))
    if drop_world:
        for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
            env.pop(k, None)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config",
                           "c1", "--steps", "3", "--warmup", "3", "--gpus", str(gpus)], capture_output=True,
                          text=True, env=env, cwd=ROOT, timeout=600)


def test_reference_arm_json_line():
    r = _run({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0"})
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("effective GFLOP/s") and d["unit"] == "GFLOP/s"
    assert d["value"] > 0 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["e2e"] == {"value": d["value"], "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["config"]["workload"].startswith("c1")


def test_reference_arm_silent_on_other_ranks():
    r = _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}, gpus=2)
    assert r.returncode == 0, r.stderr
    assert r.stdout.strip() == ""


def test_gpus_flag_without_torchrun_prints_one_line():
    """`bench.py --gpus 2` outside torchrun: the reference arm runs once (rank 0's work)
    and reports n_gpus = 2 (the native arm spawns 2 ranks itself)."""
    r = _run(gpus=2, drop_world=True)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1 and json.loads(lines[0])["n_gpus"] == 2


def test_gpus_flag_must_match_world_size():
    r = _run({"RANK": "0", "WORLD_SIZE": "2", "LOCAL_RANK": "0"}, gpus=4)
    assert r.returncode != 0 and "disagrees" in r.stderr


def test_rank_images_weak_and_strong():
    """bench.py's batch per rank: weak = the config's batch on every rank (disjoint image
    indices of the counter stream), strong = contiguous shards covering the batch once."""
    sys.path.insert(0, ROOT)
    import bench
    assert bench.rank_images(32, 4, 2, "weak") == (64, 96, 128)
    shards = [bench.rank_images(256, 8, r, "strong") for r in range(8)]
    assert [s[:2] for s in shards] == [(32 * r, 32 * r + 32) for r in range(8)] and shards[0][2] == 256
    shards = [bench.rank_images(7, 3, r, "strong")[:2] for r in range(3)]
    assert shards == [(0, 3), (3, 5), (5, 7)]
