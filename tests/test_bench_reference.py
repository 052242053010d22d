"""bench.py's reference arm (the oracle) keeps the driver's
contract on CPU: one JSON line with impl=reference and the arm's metric /
config, rank 0 only under a multi-rank launch, the weak-scaling workload of our
arm at N > 1."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(extra_env, *args):
    env = dict(os.environ, **extra_env)
    env.pop("CUDA_VISIBLE_DEVICES", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0", *args], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    out = run({})
    assert len(out) == 1
    d = json.loads(out[0])
    assert d["impl"] == "reference" and d["unit"] == "GFLOP/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["config"]["m"] == 500


def test_reference_arm_ranks():
    assert run({"RANK": "1", "WORLD_SIZE": "2"}, "--gpus", "2") == []
    d = json.loads(run({"RANK": "0", "WORLD_SIZE": "2"}, "--gpus", "2")[0])
    assert d["n_gpus"] == 2 and d["config"]["n"] == round(500 * 2 ** (1 / 3))
