"""The multi-GPU row-stripe protocol (paper_1606_00310_b200.stripes) run by
real processes over torch.distributed/gloo on CPU, with the CPU oracle as the
per-stripe compute. The gathered lattice and the combined exact moments must
equal the single-lattice oracle run (the partition-independence the
reference guarantees across worker counts, engine_vec.hpp:141-144)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, X, Y, seed, pq, mcs, out):
    import sys
    for p in (ROOT, os.path.join(ROOT, "oracle")):
        if p not in sys.path:
            sys.path.insert(0, p)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import Oracle, OracleStripe
    from paper_1606_00310_b200 import UpdateParams
    from paper_1606_00310_b200.stripes import DistTransport, StripeGroup, stripe_bounds

    o = Oracle()
    y0, y1 = stripe_bounds(Y, world, rank)
    eng = OracleStripe(o, X, Y, y0, y1, seed)
    grp = StripeGroup(DistTransport(eng, lambda nb: torch.zeros(nb, dtype=torch.uint8)), X, Y)
    prm = UpdateParams.make(*pq)
    grp.step(prm, mcs)
    rec = grp.measure()
    parts = [None] * world
    dist.all_gather_object(parts, (y0, eng.planes(), eng.states()))
    if rank == 0:
        out.put((parts, rec.power_sums, rec.mean_h, rec.W2))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,X,Y,pq,mcs", [
    (2, 256, 34, (0.5, 0.0), 6),
    (3, 384, 40, (0.75, 0.25), 5),
    (2, 128, 12, (0.98, 0.02), 3),
    (2, 256, 66, (1.0, 0.0), 4),
])
def test_stripes_over_gloo_match_single_lattice(oracle, world, X, Y, pq, mcs):
    from oracle import OracleLattice

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, X, Y, 11, pq, mcs, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue as _q
    import time
    deadline = time.time() + 300
    while True:
        try:
            parts, sums, mean, W2 = q.get(timeout=1)
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
    L = OracleLattice.flat(oracle, X, Y, 11)
    L.step(oracle, oracle.resolve(pq[0]), oracle.resolve(pq[1]), mcs)
    assert np.array_equal(planes, L.planes)
    assert np.array_equal(states, L.states)
    h, err = oracle.reconstruct(L.planes)
    assert err is None
    assert list(sums) == oracle.power_sums(h)
    assert mean == oracle.height_moments(h)[0]


def test_stripe_bounds_follow_sweep_plan():
    from paper_1606_00310_b200.stripes import stripe_bounds
    # SweepPlan::make(10, 3): base 3, remainder 1 to the last block
    assert [stripe_bounds(10, 3, i) for i in range(3)] == [(0, 3), (3, 6), (6, 10)]
    assert [stripe_bounds(8, 2, i) for i in range(2)] == [(0, 4), (4, 8)]
    assert stripe_bounds(1 << 17, 8, 7) == (7 << 14, 8 << 14)


def test_combine_reproduces_global_moments(oracle):
    """Binomial shift of stripe-local exact sums == global sums (no GPU)."""
    from oracle import OracleLattice, OracleStripe
    from paper_1606_00310_b200.stripes import StripeMoments, combine

    X, Y = 256, 30
    L = OracleLattice.flat(oracle, X, Y, 3)
    L.step(oracle, oracle.resolve(0.5), oracle.resolve(0.0), 20)
    parts = []
    for (y0, y1) in [(0, 7), (7, 19), (19, 30)]:
        st = OracleStripe(oracle, X, Y, y0, y1, 3)
        st.buf[:, st.HA:st.HA + y1 - y0] = L.planes[:, y0:y1]
        parts.append(st.measure_local())
    rec = combine(parts, X, Y)
    h, _ = oracle.reconstruct(L.planes)
    assert list(rec.power_sums) == oracle.power_sums(h)
    m = oracle.height_moments(h)
    assert rec.mean_h == m[0]
    assert abs(rec.W2 - m[1]) <= X * Y * 2.0 ** -52 * m[1]
    # serialisation used by the all_gather
    for p in parts:
        assert StripeMoments.from_array(p.to_array()) == p
