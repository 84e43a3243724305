"""N>1 path on CPU: two processes (gloo, world_size 2) shard replicas p mod 2 exactly as
bench.py does on GPUs, each computes its shard (here with the oracle — the CPU stand-in for
the per-GPU kernel), and the single end-of-run all-gather (paper_2203_09353_b200.dist)
reassembles finals in procedure order. The result must equal a single-process run bitwise."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, procedures, out_q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    from oracle_lib import McCfg, Oracle
    from paper_2203_09353_b200.dist import gather_finals, shard_procedures

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    cfg = McCfg(spins=6, steps=50, seed=5)
    mine = shard_procedures(procedures, rank, world)
    finals = []
    for p in mine:
        _, ent, _, _, _, _ = o.mc_procedure(cfg, int(p))
        finals.append(ent[-1])
    all_finals, avg, best, best_e = gather_finals(np.array(finals), procedures, rank, world)
    out_q.put((rank, all_finals, avg, best, best_e))
    dist.destroy_process_group()


@pytest.mark.parametrize("procedures", [7, 8])
def test_two_rank_shard_and_gather(procedures, oracle):
    from oracle_lib import McCfg
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, procedures, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = oracle.run(McCfg(spins=6, steps=50, seed=5), 0, procedures)
    want = single.entropies[:, -1]
    want_avg = 0.0
    for x in want:
        want_avg += float(x)
    want_avg /= procedures
    for rank, finals, avg, best, best_e in results:
        assert np.array_equal(finals.view(np.uint64), want.view(np.uint64))
        assert avg == want_avg
        assert best == int(np.argmax(want)) and best_e == float(want.max())


def test_shard_partition():
    from paper_2203_09353_b200.dist import shard_procedures
    for n in (1, 5, 64, 4096):
        for world in (1, 2, 3, 8):
            parts = [shard_procedures(n, r, world) for r in range(world)]
            allp = np.sort(np.concatenate(parts))
            assert np.array_equal(allp, np.arange(n))
            for r, part in enumerate(parts):
                assert (part % world == r).all()
