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


def test_byte_model_matches_the_scope_table():
    """bench.py's algorithmic bytes per iteration against the figures SURVEY.md 8(d) prints for
    the configs (B_spmv and B(p) at the table's average p): c3 83.8 MB / 2.600 GB, c4 1.740 GB /
    15.16 GB, c5 (int64 columns and row pointers) 18.23 GB / 125.6 GB; and the ideal it/s at
    8 TB/s the table derives from them (c3 3,076; c4 528)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", BENCH)
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    cases = {  # n, nnz, average p of the table, s_col, s_ptr, B_spmv, B(p)
        "c3": (1024 ** 2, 5238784, 150, 4, 4, 83.8e6, 2.600e9),
        "c4": (256 ** 3, 117047296, 50, 4, 4, 1.740e9, 15.16e9),
        "c5": (512 ** 3, 937951232, 50, 8, 8, 18.23e9, 125.6e9),
    }
    for name, (n, nnz, p, sc, sp, b_spmv, b_p) in cases.items():
        assert abs(bench.byte_model(n, nnz, 0, sc, sp) - b_spmv) <= 6e-4 * b_spmv, name
        assert abs(bench.byte_model(n, nnz, p, sc, sp) - b_p) <= 6e-4 * b_p, name
    assert round(8e12 / bench.byte_model(1024 ** 2, 5238784, 150)) in range(3070, 3082)
    assert round(8e12 / bench.byte_model(256 ** 3, 117047296, 50)) in range(526, 530)
    # the bench's step: one GMRES(100) cycle, p = 1..100
    n, nnz = 256 ** 3, 117047296
    assert bench.cycle_avg_bytes(n, nnz) == sum(bench.byte_model(n, nnz, p) for p in range(1, 101)) / 100
    assert bench.bench_config(2, 1)["nnz"] == nnz and bench.bench_config(2, 1)["n"] == n
