"""World-size-2 coverage of the N>1 bench path on CPU (gloo).

Each rank runs its own executor shard over the same request stream shape
(weak scaling, no data-path collective); the process group only carries the
barrier and the max-over-ranks time, exactly as bench.py does under torchrun.
Oracle executors stand in for the GPUs here."""

import json
import os
import socket
import subprocess
import sys
import textwrap

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = textwrap.dedent(r'''
import json, os, sys, time
sys.path.insert(0, os.environ["KAAS_ROOT"])
import bench
from oracle.executor import DictStore, OracleExecutor
from paper_2212_08146_b200 import workloads as W

rank, world, local, dist = bench.init_dist()
store = DictStore()
W.seed_jacobi(store, 64, prefix="j")
ex = OracleExecutor(1 << 24, store)
t0 = time.perf_counter()
oks = 0
for i in range(5):
    r = ex.execute(W.jacobi_request(f"r{rank}/{i}", 64, 10, "j/A/64", "j/b/64", "j/x0/64",
                                    f"j/x{rank}", f"j/r{rank}"))
    oks += r.status.ok
el = time.perf_counter() - t0
bench.barrier(dist)
mx = bench.allreduce_max(dist, el + rank)  # rank 1 reports +1 s: max must see it
print(json.dumps({"rank": rank, "world": world, "oks": oks, "max": mx, "mine": el}))
dist.destroy_process_group()
''')


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def test_two_rank_gloo_shards_and_max_over_ranks(tmp_path):
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), KAAS_ROOT=ROOT,
                   CUDA_VISIBLE_DEVICES="")
        procs.append(subprocess.Popen([sys.executable, str(script)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=300)
        assert p.returncode == 0, err
        outs.append(json.loads(out.strip().splitlines()[-1]))
    assert {o["rank"] for o in outs} == {0, 1}
    assert all(o["world"] == 2 and o["oks"] == 5 for o in outs)
    mx = max(o["mine"] + o["rank"] for o in outs)
    assert all(abs(o["max"] - mx) < 1e-9 for o in outs)
