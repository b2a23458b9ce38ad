"""Multi-process plumbing of the multi-GPU path on CPU (gloo, world size 2):
the NCCL unique id travels from rank 0 over the torch process group exactly as
bench.py does it, and the max-over-ranks timing reduction used by bench.py."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_2108_11932_b200 import tlr
    try:
        uid = tlr.nccl_unique_id() if rank == 0 else None
    except Exception as e:  # NCCL library absent: the id is still plain bytes
        uid = b"\x00" * 128 if rank == 0 else None
        q.put(("nccl", str(e)))
    obj = [uid]
    dist.broadcast_object_list(obj, src=0)
    t = bench.allmax(dist, 1.0 + rank)
    q.put((rank, obj[0], t))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_id_broadcast_and_allmax_over_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = {}
    while not q.empty():
        item = q.get()
        if item[0] != "nccl":
            got[item[0]] = item[1:]
    assert set(got) == {0, 1}
    assert got[0][0] == got[1][0] and len(got[0][0]) == 128
    assert got[0][1] == got[1][1] == 2.0


def test_bench_torchrun_contract_reference_arm_world2():
    """bench.py launched the way the driver launches N > 1 (torch.distributed.run,
    two ranks, 127.0.0.1): rank 0 alone runs the reference arm and prints ONE
    JSON line, the other rank exits 0 without work."""
    import json
    import subprocess
    import sys
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OPENBLAS_NUM_THREADS="1", TLRG_REF_BUDGET_S="60")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--impl", "reference", "--config", "cfg1", "--gpus", "2", "--steps", "1",
           "--warmup", "0"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
