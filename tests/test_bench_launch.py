"""bench.py's launcher (CPU): `bench.py --gpus N` run as a plain command re-executes itself
under torch.distributed.run with N ranks, and the lines report the world size measured."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out):
    res = []
    for ln in out.splitlines():
        ln = ln.strip()
        if ln.startswith("{"):
            res.append(json.loads(ln))
    return res


def _run(*args, timeout=300):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=timeout)
    return p.returncode, _lines(p.stdout), p.stderr


def test_plain_gpus_2_spawns_two_ranks():
    rc, lines, err = _run("--gpus", "2", "--launch-check")
    assert rc == 0, err
    assert sorted(x["rank"] for x in lines) == [0, 1]
    assert all(x["world"] == 2 and x["relaunched"] for x in lines)


def test_single_gpu_is_not_relaunched():
    rc, lines, err = _run("--gpus", "1", "--launch-check")
    assert rc == 0, err
    assert lines == [{"rank": 0, "world": 1, "relaunched": False}]


def test_reference_arm_reports_world_size():
    """--impl reference under the launcher: rank 0 alone prints one line, n_gpus = 2."""
    rc, lines, err = _run("--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0",
                          "--workload", "config1")
    assert rc == 0, err
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"]["parallelism"] == "crop-sharded dp2"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
