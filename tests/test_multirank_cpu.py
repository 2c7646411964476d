"""The sharded (N>1) path's host logic with world_size 2 over gloo on CPU.

On the GPU box the engine block-shards chains over ranks, each rank pre-sums
its chains' raw moments, an NCCL all-reduce pools them, and every rank
applies the merge weights (proj/src/moments.cpp:51-75); PSRF inputs are
all-gathered. Here the same host functions of libdiam.so (diamx_shard_range,
diamx_merge_weights, diamx_psrf_max) drive a gloo all-reduce / all-gather
between two processes, and the result must equal the oracle's single-process
merge_batch over all chains in ascending order (to summation-order rounding,
1e-12 as proj/tests/test_moments.cpp:184-195) and its PSRF.
"""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

P, D, PER_CHAIN, NG = 5, 6, 40, 120


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def chain_data():
    rng = np.random.default_rng(7)
    means, seconds, samples = [], [], []
    for p in range(P):
        x = rng.normal(size=(PER_CHAIN, D)) * (1 + p) + p
        samples.append(x)
        means.append(x.mean(axis=0))
        seconds.append(x.T @ x / PER_CHAIN)
    g = rng.normal(size=(NG, D))
    return means, seconds, g.mean(axis=0), g.T @ g / NG


def worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1506_05741_b200 as pkg
    lib = pkg.load().lib
    first, count = C.c_int64(), C.c_int64()
    lib.diamx_shard_range.argtypes = [C.c_int64, C.c_int, C.c_int, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    lib.diamx_shard_range(P, world, rank, C.byref(first), C.byref(count))
    means, seconds, gm, gs = chain_data()
    mine = range(first.value, first.value + count.value)
    buf = torch.zeros(D * D + D, dtype=torch.float64)
    for p in mine:
        buf[: D * D] += torch.from_numpy(seconds[p].ravel())
        buf[D * D:] += torch.from_numpy(means[p])
    dist.all_reduce(buf)
    keep, wp = C.c_double(), C.c_double()
    lib.diamx_merge_weights.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_double),
                                        C.POINTER(C.c_double)]
    lib.diamx_merge_weights(NG, P, PER_CHAIN, C.byref(keep), C.byref(wp))
    S = keep.value * gs + wp.value * buf[: D * D].numpy().reshape(D, D)
    m = keep.value * gm + wp.value * buf[D * D:].numpy()
    # PSRF inputs: per-chain (mean, diag) gathered from uneven shards (pad to the largest)
    maxc = (P + world - 1) // world
    loc = torch.zeros(2 * maxc * D, dtype=torch.float64)
    for i, p in enumerate(mine):
        loc[i * D:(i + 1) * D] = torch.from_numpy(means[p])
        loc[(maxc + i) * D:(maxc + i + 1) * D] = torch.from_numpy(np.diag(seconds[p]).copy())
    gathered = [torch.zeros_like(loc) for _ in range(world)]
    dist.all_gather(gathered, loc)
    cm, cd = [], []
    for r in range(world):
        f, c = C.c_int64(), C.c_int64()
        lib.diamx_shard_range(P, world, r, C.byref(f), C.byref(c))
        g = gathered[r].numpy()
        for i in range(c.value):
            cm.append(g[i * D:(i + 1) * D])
            cd.append(g[(maxc + i) * D:(maxc + i + 1) * D])
    cm = np.ascontiguousarray(np.array(cm))
    cd = np.ascontiguousarray(np.array(cd))
    ps = C.c_double()
    dp = C.POINTER(C.c_double)
    lib.diamx_psrf_max.argtypes = [dp, dp, C.c_int64, C.c_int64, C.c_uint64, dp]
    assert lib.diamx_psrf_max(cm.ctypes.data_as(dp), cd.ctypes.data_as(dp), P, D, PER_CHAIN, C.byref(ps)) == 0
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), S=S, m=m, psrf=ps.value, first=first.value,
             count=count.value)
    dist.destroy_process_group()


def test_sharded_merge_equals_single_process_merge(tmp_path):
    world = 2
    mp.spawn(worker, args=(world, free_port(), str(tmp_path)), nprocs=world, join=True)
    import _oracle as O
    means, seconds, gm, gs = chain_data()

    class Mom(C.Structure):
        _fields_ = [("dim", C.c_size_t), ("count", C.c_uint64), ("mean", C.POINTER(C.c_double)),
                    ("second", C.POINTER(C.c_double))]

    keep_arrays = []

    def mom(mean, sec, cnt):
        a, b = np.ascontiguousarray(mean.copy()), np.ascontiguousarray(sec.copy())
        keep_arrays.extend([a, b])
        return Mom(D, cnt, O.dptr(a), O.dptr(b))

    glob = mom(gm, gs, NG)
    locals_ = (Mom * P)(*[mom(means[p], seconds[p], PER_CHAIN) for p in range(P)])
    batches = C.c_uint64(0)
    L = O.oracle()
    L.or_merge_batch.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p, C.c_size_t]
    assert L.or_merge_batch(C.byref(glob), C.byref(batches), locals_, P) == 0
    S_ref = np.ctypeslib.as_array(glob.second, shape=(D * D,)).reshape(D, D).copy()
    m_ref = np.ctypeslib.as_array(glob.mean, shape=(D,)).copy()
    L.or_psrf_max.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_double)]
    psrf_ref = C.c_double()
    assert L.or_psrf_max(locals_, P, C.byref(psrf_ref)) == 0
    covered = []
    for r in range(world):
        z = np.load(tmp_path / f"rank{r}.npz")
        covered += list(range(int(z["first"]), int(z["first"]) + int(z["count"])))
        assert np.linalg.norm(z["S"] - S_ref) / np.linalg.norm(S_ref) < 1e-12
        assert np.linalg.norm(z["m"] - m_ref) / np.linalg.norm(m_ref) < 1e-12
        assert abs(float(z["psrf"]) - psrf_ref.value) < 1e-12
    assert sorted(covered) == list(range(P))  # every chain owned exactly once
