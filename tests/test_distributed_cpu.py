"""N > 1 host path on CPU: sharding and the single allreduce of the average
numerator, world_size 2 over gloo (127.0.0.1), checked against the serial sum
of the oracle's rotate_expansion (src/steer.cpp:208-223)."""
import math
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2509_01180_b200.distributed import allreduce_average, shard_range


def test_shard_range_covers_all():
    for n in (0, 1, 7, 1024, 131072):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    from oracle import bmo
    spec = bmo.Spec(6, 6 * math.pi)
    rng = np.random.default_rng(3)
    coeffs, quats = [], []
    for p in range(5):
        v = rng.standard_normal((16, 16, 16))
        coeffs.append(bmo.expand(v, spec))
        quats.append(bmo.haar_rotation(11, p))
    return spec, coeffs, quats


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from oracle import bmo
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec, coeffs, quats = _inputs()
    b, e = shard_range(len(coeffs), rank, world)
    part = np.zeros(spec.coeff_count, dtype=np.complex128)
    for p in range(b, e):
        q = quats[p]
        part += bmo.rotate_expansion(coeffs[p], spec, [q[0], -q[1], -q[2], -q[3]])
    t = torch.from_numpy(np.ascontiguousarray(np.stack([part.real, part.imag], -1)))
    avg, total = allreduce_average(t, e - b)
    out[rank] = (avg.numpy().copy(), total)
    dist.destroy_process_group()


def test_two_rank_average_allreduce_gloo():
    spec, coeffs, quats = _inputs()
    ref = np.zeros(spec.coeff_count, dtype=np.complex128)
    for c, q in zip(coeffs, quats):
        ref += bmo_rotate(spec, c, q)
    ref /= len(coeffs)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
        for r in range(2):
            avg, total = out[r]
            assert total == len(coeffs)
            got = avg[..., 0] + 1j * avg[..., 1]
            assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def bmo_rotate(spec, c, q):
    from oracle import bmo
    return bmo.rotate_expansion(c, spec, [q[0], -q[1], -q[2], -q[3]])


def _chunk_worker(rank, world, port, out):
    import torch.distributed as dist
    from oracle import bmo
    from paper_2509_01180_b200.distributed import ChunkScheduler
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    spec, coeffs, quats = _inputs()
    import torch
    part = np.zeros(spec.coeff_count, dtype=np.complex128)
    got, count = [], 0
    for b, e in ChunkScheduler(len(coeffs), 2, key="test_chunks"):
        got.append((b, e))
        for p in range(b, e):
            q = quats[p]
            part += bmo.rotate_expansion(coeffs[p], spec, [q[0], -q[1], -q[2], -q[3]])
            count += 1
    t = torch.from_numpy(np.ascontiguousarray(np.stack([part.real, part.imag], -1)))
    avg, total = allreduce_average(t, count)
    out[rank] = (got, avg.numpy().copy(), total)
    dist.destroy_process_group()


def test_two_rank_dynamic_chunks_gloo():
    """Chunks pulled from the store's atomic counter: every particle is aligned by
    exactly one rank, and the allreduced average equals the serial one."""
    spec, coeffs, quats = _inputs()
    ref = np.zeros(spec.coeff_count, dtype=np.complex128)
    for c, q in zip(coeffs, quats):
        ref += bmo_rotate(spec, c, q)
    ref /= len(coeffs)
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_chunk_worker, args=(2, port, out), nprocs=2, join=True)
        spans = sorted(s for r in range(2) for s in out[r][0])
        covered = [p for b, e in spans for p in range(b, e)]
        assert covered == list(range(len(coeffs)))
        for r in range(2):
            _, avg, total = out[r]
            assert total == len(coeffs)
            got = avg[..., 0] + 1j * avg[..., 1]
            assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def test_chunk_scheduler_single_process():
    from paper_2509_01180_b200.distributed import ChunkScheduler
    assert list(ChunkScheduler(7, 3, store=None)) == [(0, 3), (3, 6), (6, 7)]
    assert list(ChunkScheduler(0, 3, store=None)) == []
