"""bench.py launch contract on the CPU box (no GPU work): `--gpus N` without a launcher
starts N ranks itself (torch.distributed.run, rendezvous on 127.0.0.1), and under a launcher
the world size must equal --gpus."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env():
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        env.pop(k, None)
    return env


def test_gpus_n_spawns_n_ranks():
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--dry-run"], env=_env(), capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["dry_run"] and line["gpus"] == 2 and line["world"] == 2
    assert sorted(x["rank"] for x in line["ranks"]) == [0, 1]
    assert all(x["world"] == 2 for x in line["ranks"])
    assert len({x["pid"] for x in line["ranks"]}) == 2          # two processes
    assert "launching 2 ranks" in r.stderr


def test_single_rank_dry_run_does_not_relaunch():
    r = subprocess.run([sys.executable, BENCH, "--gpus", "1", "--dry-run"],
                       env=dict(_env(), MASTER_ADDR="127.0.0.1", MASTER_PORT="29581", WORLD_SIZE="1", RANK="0"),
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["world"] == 1 and "launching" not in r.stderr


def test_world_size_must_match_gpus():
    env = dict(_env(), WORLD_SIZE="3", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--dry-run"], env=env, capture_output=True,
                       text=True, timeout=120)
    assert r.returncode == 2
    assert "WORLD_SIZE=3 but --gpus 2" in r.stderr
