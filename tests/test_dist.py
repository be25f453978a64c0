"""Request-level data parallelism on CPU (gloo, world size 2): sharding, statistics reductions and
sharding invariance of per-request outputs (test tier T5)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2601_23278_b200 import dist as D


def test_shard_requests_partition_and_balance():
    for n, w in [(256, 8), (64, 2), (10, 4), (3, 4)]:
        shards = [D.shard_requests(n, w, r) for r in range(w)]
        assert sorted(sum(shards, [])) == list(range(n))
        assert max(map(len, shards)) - min(map(len, shards)) <= 1
    costs = [256 + 37 * ((i * 7919) % 113) for i in range(256)]          # mixed prompt lengths
    shards = [D.shard_requests(256, 8, r, costs) for r in range(8)]
    assert sorted(sum(shards, [])) == list(range(256))
    assert {len(s) for s in shards} == {32}
    loads = [sum(costs[i] for i in s) for s in shards]
    assert max(loads) / min(loads) < 1.02                               # LPT with equal counts
    assert shards == [D.shard_requests(256, 8, r, costs) for r in range(8)]   # deterministic


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    r, w, _ = D.init("gloo")
    assert (r, w) == (rank, world) and dist.is_initialized()
    # statistics reductions used by bench.py
    mx = D.reduce_max(float(10 + rank))
    sm = D.reduce_sum(float(rank + 1))
    st = D.all_gather_stats([rank, 7 * rank])
    # per-request decode with the CPU oracle on this rank's shard (C1-sized requests)
    from oracle.engine import OracleEngine, request_prompts
    from synth import get_config
    run = get_config("C1").with_(n_requests=5)
    prompts = request_prompts(run)
    mine = D.shard_requests(run.n_requests, world, rank)
    eng = OracleEngine(run, "gpu")
    local = {}
    for g in mine:
        eng.kv_append(g, prompts[g], run.gen_len)
        while not eng.req[g].finished:
            eng.step_one(g)
            eng.commit_one(g)
        local[g] = eng.req[g].output
    outs = D.gather_outputs(local)
    D.barrier()
    q.put((rank, mx, sm, st, outs))
    dist.destroy_process_group()


def test_world_size_2_gloo_stats_and_sharding_invariance():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, mx, sm, st, outs in res:
        assert mx == 11.0 and sm == 3.0
        assert st == [[0, 0], [1, 7]]
    assert res[0][4] == res[1][4]
    # single-process reference: the same requests decoded in one process
    from oracle.engine import run_to_completion
    from synth import get_config
    eng, _ = run_to_completion(get_config("C1").with_(n_requests=5), "gpu")
    assert res[0][4] == {g: eng.req[g].output for g in range(5)}
