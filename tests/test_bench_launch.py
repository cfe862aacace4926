"""CPU checks of bench.py's multi-GPU launch contract: `--gpus N` run directly re-launches
itself under torchrun with N ranks (rendezvous on 127.0.0.1), and a launch whose process
count differs from --gpus fails instead of measuring fewer GPUs."""
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _env(**kw):
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "P3S_BENCH_RELAUNCHED")}
    env.update(kw)
    return env


def test_gpus_n_relaunches_n_ranks():
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--launch-selftest"],
                       capture_output=True, text=True, timeout=300, env=_env())
    assert r.returncode == 0, r.stderr[-2000:]
    # both ranks share torchrun's stdout pipe: pick the records out by pattern, since a
    # line of one rank may be split by the other's
    ranks = [json.loads(m) for m in re.findall(r'\{"rank": \d+, "world": \d+, "local": \d+\}', r.stdout)]
    assert sorted(d["rank"] for d in ranks) == [0, 1]
    assert all(d["world"] == 2 for d in ranks)


def test_world_mismatch_is_an_error():
    r = subprocess.run([sys.executable, BENCH, "--gpus", "2", "--steps", "3"],
                       capture_output=True, text=True, timeout=300,
                       env=_env(P3S_BENCH_RELAUNCHED="1"))
    assert r.returncode != 0
    assert "--gpus 2 but 1 process(es)" in r.stderr


def test_torchrun_argv_and_numa_helpers():
    from paper_2009_09501_b200.sharding import node_cpus, torchrun_argv
    argv = torchrun_argv(4, "bench.py", ["--steps", "5"], port=29511)
    assert "--nproc-per-node=4" in argv and "--master-addr=127.0.0.1" in argv
    assert argv[-3:] == ["bench.py", "--steps", "5"]
    assert node_cpus(-1) == set()
    cpus = node_cpus(0)
    assert not cpus or all(isinstance(c, int) for c in cpus)
