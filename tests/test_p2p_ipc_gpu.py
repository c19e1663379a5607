"""The device-side halo exchange across PROCESSES: two ranks (spawned
processes, gloo only for the one-time CUDA IPC handle exchange and the
moment gather) each own a row stripe on the same B200, map the neighbour's
planes / counters with cudaIpcOpenMemHandle and step with no host
synchronisation between passes (csrc/p2p.cu). The gathered lattice must equal
the single periodic engine bit-exactly. On a multi-GPU node the same code runs
one rank per GPU over NVLink."""
import os
import queue as _q
import socket
import time

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, Y, seed, pq, mcs, out, fused="1"):
    import sys
    if ROOT not in sys.path:
        sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ["OCTGPU_DEEP"] = "2"  # multi-MCS passes at test sizes (constant xi)
    os.environ["OCTGPU_FUSED_LINK"] = fused  # the one-launch passes of separate GPUs, or the three launches
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1606_00310_b200 as octgpu
    from paper_1606_00310_b200.stripes import PeerDistTransport, StripeEngine, StripeGroup, stripe_bounds

    torch.cuda.set_device(0)
    cfg = octgpu.LatticeConfig(X, Y)
    y0, y1 = stripe_bounds(Y, world, rank)
    eng = StripeEngine(cfg, y0, y1, seed, device=0)
    tr = PeerDistTransport(eng)
    grp = StripeGroup(tr, X, Y)
    prm = octgpu.UpdateParams.make(*pq)
    grp.step(prm, mcs)
    rec = grp.measure()
    parts = [None] * world
    dist.all_gather_object(parts, (y0, eng.planes(), eng.states()))
    if rank == 0:
        out.put((parts, rec.power_sums))
    tr.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,X,Y,pq,mcs", [(2, 2048, 256, (1.0, 0.0), 7), (2, 1024, 200, (0.5, 0.0), 5),
                                              (3, 1024, 300, (0.75, 0.25), 4)])
@pytest.mark.parametrize("fused", ["1", "0"])
def test_peer_exchange_across_processes(world, X, Y, pq, mcs, fused):
    import paper_1606_00310_b200 as octgpu

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, Y, 13, pq, mcs, q, fused)) for r in range(world)]
    for p in procs:
        p.start()
    deadline = time.time() + 240
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
    planes = np.concatenate([pl for (_, pl, _) in parts], axis=1)
    states = np.concatenate([st for (_, _, st) in parts], axis=0)
    ref = octgpu.GpuEngine(octgpu.LatticeConfig(X, Y), 13)
    ref.step(octgpu.UpdateParams.make(*pq), mcs)
    assert np.array_equal(planes, ref.planes())
    assert np.array_equal(states, ref.streams().states)
    assert sums == ref.measure().power_sums
