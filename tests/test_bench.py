"""bench.py's host-side contract on CPU: --gpus N starts N ranks itself,
the reference arm runs from the oracle alone (no product package), and the
oracle's row-wise weight draws equal init_params."""
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra=None, timeout=600):
    env = dict(os.environ, PYTHONPATH=ROOT, RECMG_DIST_BACKEND="gloo",
               OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-3000:]
    return json.loads(lines[0]), out


SMALL = ["--impl", "reference", "--accesses", "300000", "--tables", "16", "--rows", "2000",
         "--cpu-sample", "3000", "--steps", "1", "--warmup", "0"]


def test_gpus_flag_spawns_ranks_and_reference_arm_is_oracle_only():
    line, _ = _run(["--gpus", "2", "--config", "2"] + SMALL)
    assert line["n_gpus"] == 2 and line["impl"] == "reference"
    assert line["cpu_baseline"]["kind"] == "port"
    # the reference arm never imports the product package
    code = ("import runpy, sys; sys.argv = ['bench.py'] + %r; "
            "sys.modules['paper_2511_08568_b200'] = None; "
            "runpy.run_path('bench.py', run_name='__main__')" % (SMALL,))
    env = dict(os.environ, PYTHONPATH=ROOT)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    one = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert one["config"] == line["config"]


def test_config3_default_for_several_ranks_and_sharded_reference():
    """N > 1 defaults to config 3 (table-sharded, strong scaling); the
    reference arm shards its oracle-generated trace the same way."""
    line, _ = _run(["--gpus", "2", "--impl", "reference", "--accesses", "400000",
                    "--tables", "24", "--rows", "3000", "--cpu-sample", "3000", "--steps", "1",
                    "--warmup", "0"])
    assert line["n_gpus"] == 2 and line["scaling"] == "strong"
    assert line["config"]["workload"].startswith("config3") and line["config"]["shards"] == 2
    assert "shard 0 sub-trace of config 3" in line["cpu_baseline"]["sample"]


def test_oracle_row_draws_equal_init_params():
    from oracle import cpu_baseline as cb
    from oracle import model_oracle as mo
    sizes = [30, 7, 50]
    for kind, seed in (("caching", 0), ("prefetch", 1)):
        full = mo.init_arrays(kind, sizes, 8, seed=seed, init_scale=0.4)
        rows = np.array([0, 5, 36, 86])
        got, _ = cb.draw_params(kind, sizes, 8, rows, seed, 0.4)
        assert np.array_equal(got["embed_id"], full["embed_id"][rows])
        for k, v in full.items():
            if k != "embed_id":
                assert np.array_equal(got[k], v), k
