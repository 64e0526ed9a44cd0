#!/usr/bin/env python3
"""Build compile-time variants of libigs.so side by side (vars/<name>/, git-ignored) for A/B
timing on the GPU box:  python tools/variants.py build name1='-DX=1' name2='-DX=2' ...
then on the box:        python tools/variants.py run --config c2 --alg igs2 name1 name2 ...
Each variant is a copy of the package + include + workloads + tools/bench_configs.py."""
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build(specs):
    for spec in specs:
        name, flags = spec.split("=", 1)
        d = os.path.join(ROOT, "vars", name)
        shutil.rmtree(d, ignore_errors=True)
        os.makedirs(os.path.join(d, "tools"))
        for sub in ("paper_2205_07805_b200", "include", "workloads"):
            shutil.copytree(os.path.join(ROOT, sub), os.path.join(d, sub),
                            ignore=shutil.ignore_patterns("*.so", "__pycache__"))
        shutil.copy(os.path.join(ROOT, "tools", "bench_configs.py"), os.path.join(d, "tools"))
        env = dict(os.environ, IGS_NVCC_EXTRA=flags)
        subprocess.run([sys.executable, "-c", "from paper_2205_07805_b200 import build; build.build(force=True)"],
                       cwd=d, env=env, check=True)
        print("built", name, flags)


def run(args):
    names = [a for a in args if not a.startswith("--")]
    opts = [a for a in args if a.startswith("--")]
    extra = []
    for o in opts:
        extra += o.split("=", 1)
    for name in names:
        d = os.path.join(ROOT, "vars", name)
        r = subprocess.run([sys.executable, "tools/bench_configs.py", *extra], cwd=d, capture_output=True,
                           text=True, env=dict(os.environ, IGS_PC_PROF="1"))
        prof = [l for l in r.stderr.splitlines() if "pcycle" in l]
        print(name, (prof[-1] if prof else ""), r.stdout.strip().splitlines()[-1][:220] if r.stdout.strip() else r.stderr[-400:])


if __name__ == "__main__":
    {"build": build, "run": run}[sys.argv[1]](sys.argv[2:])
