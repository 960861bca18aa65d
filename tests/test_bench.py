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


def _c3_rank(rank, world, port, out):
    import torch  # noqa: F401
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, ROOT)
    import bench

    class A:
        accesses, tables, rows, dim, init_scale = 200_000, 16, 1000, 8, 0.4
        shards_eff, world, shard_index = 2, 2, 0
    st = bench.build_state_config3(A, rank, None, device=False, dist=dist)
    out[rank] = (st[0].gid_array.copy(), st[-1].tables)
    dist.barrier()
    dist.destroy_process_group()


def test_config3_trace_streamed_once_per_node_and_shared():
    """Under several ranks the config-3 trace is streamed by local rank 0 into
    /dev/shm and mapped by the others; the shards partition the trace and the
    shared copy is removed."""
    import glob
    import multiprocessing as mp
    import socket
    from paper_2511_08568_b200 import TraceGenConfig, generate_trace
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mgr = mp.Manager()
    out = mgr.dict()
    ps = [mp.Process(target=_c3_rank, args=(r, 2, port, out)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    assert all(p.exitcode == 0 for p in ps)
    full = generate_trace(TraceGenConfig([1000] * 16, 200_000, 1.05, 0.4, 32, 3)).gid_array
    (g0, t0), (g1, t1) = out[0], out[1]
    assert sorted(set(t0) | set(t1)) == list(range(16)) and not set(t0) & set(t1)
    assert len(g0) + len(g1) == len(full)
    assert np.array_equal(g0, full[np.isin(full // 1000, t0)])
    assert not glob.glob("/dev/shm/recmg_c3_16x1000_200000_*")
