"""Row stripes on DIFFERENT GPUs (BASELINE configs[4]): the partition of the reference's
SweepPlan (params.hpp:107-127) with halos exchanged (1) device-side over peer memory inside one process,
(2) across processes (one rank per GPU) over CUDA IPC peer memory, (3) across processes over NCCL
isend/irecv. Each must reproduce the single periodic engine bit-exactly. These need >= 2 visible devices
and skip otherwise (the gpurun boxes of this build have one B200; the same protocols are exercised on one
device by tests/test_stripes_gpu.py and tests/test_p2p_ipc_gpu.py)."""
import os
import queue as _q
import socket
import time

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import paper_1606_00310_b200 as octgpu
from conftest import ROOT

pytestmark = pytest.mark.gpu

NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0
need2 = pytest.mark.skipif(NDEV < 2, reason="needs >= 2 GPUs")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _reference(X, Y, seed, schedule):
    ref = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), seed, device=0)
    for pq, n in schedule:
        ref.step(octgpu.UpdateParams.make(*pq), n)
    return ref


SCHEDULE = [((1.0, 0.0), 5), ((0.5, 0.0), 3), ((0.5, 0.5), 2)]


@need2
@pytest.mark.parametrize("parts", [2, 4, 8])
def test_peer_stripes_on_several_devices_in_one_process(parts):
    """One stripe per device (round robin), device-side halo exchange over NVLink peer memory."""
    from paper_1606_00310_b200.stripes import PeerLocalTransport, StripeEngine, StripeGroup, stripe_bounds

    X, Y, seed = 2048, 1024, 5
    cfg = octgpu.LatticeConfig(X, Y)
    engines = []
    for r in range(parts):
        y0, y1 = stripe_bounds(Y, parts, r)
        engines.append(StripeEngine(cfg, y0, y1, seed, device=r % NDEV))
    grp = StripeGroup(PeerLocalTransport(engines), X, Y)
    for pq, n in SCHEDULE:
        grp.step(octgpu.UpdateParams.make(*pq), n)
    for e in engines:
        e.sync()
    ref = _reference(X, Y, seed, SCHEDULE)
    assert np.array_equal(np.concatenate([e.planes() for e in engines], axis=1), ref.planes())
    assert np.array_equal(np.concatenate([e.states() for e in engines], axis=0), ref.streams().states)
    assert grp.measure().power_sums == ref.measure().power_sums


def _worker(rank, world, port, transport, X, Y, seed, out):
    import sys
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl" if transport == "nccl" else "gloo", rank=rank, world_size=world)
    import paper_1606_00310_b200 as octgpu
    from paper_1606_00310_b200.stripes import (DistTransport, PeerDistTransport, StripeEngine, StripeGroup,
                                               stripe_bounds)

    cfg = octgpu.LatticeConfig(X, Y)
    y0, y1 = stripe_bounds(Y, world, rank)
    eng = StripeEngine(cfg, y0, y1, seed, device=rank)
    if transport == "nccl":
        alloc = lambda nb: torch.zeros(nb, dtype=torch.uint8, device=f"cuda:{rank}")  # noqa: E731
        tr = DistTransport(eng, alloc)
    else:
        tr = PeerDistTransport(eng)
    grp = StripeGroup(tr, X, Y)
    for pq, n in SCHEDULE:
        grp.step(octgpu.UpdateParams.make(*pq), n)
    eng.sync()
    rec = grp.measure()
    parts = [None] * world
    dist.all_gather_object(parts, (y0, eng.planes(), eng.states()))
    if rank == 0:
        out.put((parts, rec.power_sums))
    if hasattr(tr, "close"):
        tr.close()
    dist.destroy_process_group()


@need2
@pytest.mark.parametrize("transport", ["ipc", "nccl"])
def test_one_rank_per_device(transport):
    world, X, Y, seed = min(NDEV, 4), 2048, 1024, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, transport, X, Y, seed, q)) for r in range(world)]
    for p in procs:
        p.start()
    deadline = time.time() + 300
    while True:
        try:
            parts, sums = q.get(timeout=1)
            break
        except _q.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() > deadline:
                for p in procs:
                    p.kill()
                pytest.fail("a rank failed: " + str([p.exitcode for p in procs]))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts.sort(key=lambda t: t[0])
    ref = _reference(X, Y, seed, SCHEDULE)
    assert np.array_equal(np.concatenate([pl for (_, pl, _) in parts], axis=1), ref.planes())
    assert np.array_equal(np.concatenate([st for (_, _, st) in parts], axis=0), ref.streams().states)
    assert sums == ref.measure().power_sums
