"""Multi-rank host logic on CPU (gloo, world_size 2): the drop sharding and the one
exchange step (combining per-rank ergodic sums/counts and saturation statistics)
reproduce the single-rank result.  The per-drop results come from the oracle
here (CPU box, no GPU); on GPUs the same combine runs over NCCL in bench.py."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2503_18118_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sweep_result(orc, pos, n_list, snr, recv, lam, gram_kind=0):
    a = orc.array("ula", n_y=max(n_list), fc_hz=28e9)
    erg, nv, sat, _, ergv = orc.saturation_sweep(a, n_list, pos, snr, recv, gram_kind=gram_kind, nthreads=1,
                                                 valid_mean=True)
    return {"ergodic": erg, "n_valid": nv, "ergodic_valid": ergv, "sat": sat}


def _worker(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as orc
    total = 36
    first, n = parallel.shard_range(total, rank, world)
    pos = orc.gen_drops(orc.users(r=(3.0, 30.0)), 4, n, seed=5, first_drop=first)
    lam = 299792458.0 / 28e9
    out = {}
    for gk in (0, 1):   # exact; closed form (cfg1-like drops with NaN ZF rates, R10)
        res = _sweep_result(orc, pos, [64, 128, 256], [0.0, 10.0], 7, lam, gram_kind=gk)
        comb = parallel.allreduce_sweep(res, n, dist, torch.device("cpu"), pitch=lam / 2)
        out[gk] = {k: np.asarray(v) for k, v in comb.items()}
    if rank == 0:
        out_q.put(out)
    dist.destroy_process_group()


def test_shard_range_partitions():
    for total in (1, 7, 10000):
        for world in (1, 2, 3, 8):
            spans = [parallel.shard_range(total, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (f0, n0), (f1, _) in zip(spans, spans[1:]):
                assert f0 + n0 == f1
            assert sum(n for _, n in spans) == total


def test_pack_unpack_single_rank_identity(orc):
    pos = orc.gen_drops(orc.users(r=(3.0, 30.0)), 4, 10, seed=2)
    lam = 299792458.0 / 28e9
    res = _sweep_result(orc, pos, [64, 128], [10.0], 7, lam)
    back = parallel.unpack_sweep(parallel.pack_sweep(res, 10, lam / 2), res["ergodic"].shape, lam / 2)
    assert np.allclose(back["ergodic"], res["ergodic"], rtol=1e-13)
    assert np.allclose(back["ergodic_valid"], res["ergodic_valid"], rtol=1e-13)
    assert np.array_equal(back["n_valid"], res["n_valid"])
    assert np.allclose(back["sat"], res["sat"], rtol=1e-10)


def test_two_rank_combine_equals_single_rank(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    comb = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    pos = orc.gen_drops(orc.users(r=(3.0, 30.0)), 4, 36, seed=5)
    lam = 299792458.0 / 28e9
    for gk in (0, 1):
        ref = _sweep_result(orc, pos, [64, 128, 256], [0.0, 10.0], 7, lam, gram_kind=gk)
        c = comb[gk]
        np.testing.assert_array_equal(np.isnan(c["ergodic"]), np.isnan(ref["ergodic"]))
        assert np.allclose(c["ergodic"], ref["ergodic"], rtol=1e-12, atol=1e-12, equal_nan=True)
        assert np.allclose(c["ergodic_valid"], ref["ergodic_valid"], rtol=1e-12, atol=1e-12, equal_nan=True)
        assert np.array_equal(c["n_valid"], ref["n_valid"])
        assert np.allclose(c["sat"][[0, 1, 3]], ref["sat"][[0, 1, 3]], rtol=1e-9)
        assert c["sat"][2] == ref["sat"][2]
        if gk == 1:
            assert np.any(ref["n_valid"] < 36)       # the strict-NaN rule is exercised across ranks
