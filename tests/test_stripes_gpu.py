"""Row stripes on the GPU: several StripeEngines on one device, exchanging
halos through the same protocol the multi-GPU path uses (LocalTransport),
must reproduce the single periodic engine bit-exactly (planes, rng states,
exact moments). This is the 1/2/4/8-GPU identity check run on one B200."""
import numpy as np
import pytest
import torch

import paper_1606_00310_b200 as octgpu
from paper_1606_00310_b200.stripes import LocalTransport, PeerLocalTransport, StripeEngine, StripeGroup, stripe_bounds

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _deep_passes_at_test_sizes(monkeypatch):
    """The 2-MCS stripe passes are the default only from 2^28 sites per stripe; force them at
    test sizes (constant-xi modes; odd MCS counts still run one-MCS passes)."""
    monkeypatch.setenv("OCTGPU_DEEP", "2")


def _group(cfg, parts, seed, stream, transport="host"):
    engines = []
    streams = []
    for r in range(parts):
        y0, y1 = stripe_bounds(cfg.Y, parts, r)
        e = StripeEngine(cfg, y0, y1, seed)
        if transport == "peer-streams":  # one stream per stripe: passes run concurrently, ordered by the counters
            streams.append(torch.cuda.Stream())
            e.set_stream(streams[-1].cuda_stream)
        else:
            e.set_stream(stream.cuda_stream)
        engines.append(e)
    if transport.startswith("peer"):
        return StripeGroup(PeerLocalTransport(engines), cfg.X, cfg.Y), engines
    alloc = lambda nb: torch.zeros(nb, dtype=torch.uint8, device="cuda")  # noqa: E731
    return StripeGroup(LocalTransport(engines, alloc), cfg.X, cfg.Y), engines


# (1024, 48, 8): 6-row stripes, the minimum (the 3-MCS pass reads 6 rows of the next stripe)
@pytest.mark.parametrize("X,Y,parts", [(1024, 128, 2), (1024, 130, 4), (2048, 96, 3), (256, 40, 2), (8192, 512, 8),
                                       (1024, 48, 8)])
@pytest.mark.parametrize("pq", [(0.5, 0.0), (0.98, 0.02), (1.0, 0.0), (0.75, 0.5), (0.0, 0.0)])
@pytest.mark.parametrize("transport", ["host", "peer", "peer-streams", "peer-fused"])
def test_stripes_match_single_engine(X, Y, parts, pq, transport, monkeypatch):
    if transport.startswith("peer") and X < 1024:
        pytest.skip("the peer-memory exchange runs the TMA kernels (X >= 1024)")
    if transport == "peer-fused":  # the one-launch passes (default only when neighbours are on other GPUs)
        monkeypatch.setenv("OCTGPU_FUSED_LINK", "1")
        transport = "peer-streams"
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        cfg = octgpu.LatticeConfig(X, Y)
        prm = octgpu.UpdateParams.make(*pq)
        grp, engines = _group(cfg, parts, 21, stream, transport)
        grp.step(prm, 7)
        for e in engines:
            e.sync()  # the per-stripe streams, and a timed-out peer wait would raise here
        ref = octgpu.GpuEngine(cfg, 21)
        ref.step(prm, 7)
        torch.cuda.synchronize()
        planes = np.concatenate([e.planes() for e in engines], axis=1)
        states = np.concatenate([e.states() for e in engines], axis=0)
        assert np.array_equal(planes, ref.planes())
        assert np.array_equal(states, ref.streams().states)
        rec, rref = grp.measure(), ref.measure()
        assert rec.power_sums == rref.power_sums
        assert rec.mean_h == rref.mean_h
        assert abs(rec.W2 - rref.W2) <= 2 ** -50 * rref.W2


@pytest.mark.parametrize("X,Y,parts", [(1024, 128, 2), (1024, 130, 4), (2048, 96, 3), (8192, 512, 8), (1024, 48, 8)])
@pytest.mark.parametrize("pq", [(0.5, 0.0), (0.5, 0.5), (0.98, 0.02), (1.0, 0.0), (0.75, 0.25)])
@pytest.mark.parametrize("transport", ["host", "peer", "peer-fused"])
def test_counter_rng_stripes_match_single_engine(X, Y, parts, pq, transport, monkeypatch):
    """Opt-in counter streams on row stripes (k_mcs_bulk<CTR> / k_mcs_deep<CTR> with local -> global rows):
    the striped run equals the periodic engine's (itself pinned to the oracle's oo_step_ctr)."""
    if transport == "peer-fused":
        monkeypatch.setenv("OCTGPU_FUSED_LINK", "1")
        transport = "peer"
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        cfg = octgpu.LatticeConfig(X, Y)
        prm = octgpu.UpdateParams.make(*pq)
        engines = []
        for r in range(parts):
            y0, y1 = stripe_bounds(Y, parts, r)
            e = StripeEngine(cfg, y0, y1, 21)
            e.set_stream(stream.cuda_stream)
            e.set_rng("counter")
            engines.append(e)
        if transport == "peer":
            grp = StripeGroup(PeerLocalTransport(engines), X, Y)
        else:
            grp = StripeGroup(LocalTransport(engines, lambda nb: torch.zeros(nb, dtype=torch.uint8, device="cuda")),
                              X, Y)
        grp.step(prm, 7)
        for e in engines:
            e.sync()
        ref = octgpu.GpuEngine(cfg, 21)
        ref.set_rng("counter")
        ref.step(prm, 7)
        torch.cuda.synchronize()
        planes = np.concatenate([e.planes() for e in engines], axis=1)
        assert np.array_equal(planes, ref.planes())
        rec, rref = grp.measure(), ref.measure()
        assert rec.power_sums == rref.power_sums


def test_stripe_curl_violation_reported_globally():
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        X, Y = 1024, 64
        cfg = octgpu.LatticeConfig(X, Y)
        ref = octgpu.GpuEngine(cfg, 5)
        ref.step(octgpu.UpdateParams.make(0.5, 0.0), 4)
        planes, states = ref.planes(), ref.streams().states
        planes[0, 40, 3] ^= np.uint64(1 << 9)  # corrupt a row owned by the second stripe
        engines = []
        for r in range(2):
            y0, y1 = stripe_bounds(Y, 2, r)
            e = StripeEngine(cfg, y0, y1, 5, planes=planes[:, y0:y1], states=states[y0:y1], t=4)
            e.set_stream(stream.cuda_stream)
            engines.append(e)
        grp = StripeGroup(LocalTransport(engines, lambda nb: torch.zeros(nb, dtype=torch.uint8, device="cuda")), X, Y)
        bad = octgpu.GpuEngine(octgpu.SlopeField(cfg, planes, 4, 0), octgpu.RngStreamSet(5, states))
        with pytest.raises(octgpu.InvariantError) as e1:
            bad.measure()
        with pytest.raises(octgpu.InvariantError) as e2:
            grp.measure()
        assert str(e1.value) == str(e2.value)


def test_stripe_pass_sizes():
    cfg = octgpu.LatticeConfig(1024, 64)
    e = StripeEngine(cfg, 0, 32, 3)
    assert e.max_mcs(octgpu.UpdateParams.make(1.0, 0.0)) == 3  # constant xi: 3-MCS passes (k_mcs_deep)
    assert e.max_mcs(octgpu.UpdateParams.make(0.5, 0.0)) == 1
    assert e.pass_plan(octgpu.UpdateParams.make(1.0, 0.0)) == ("k_mcs_deep", 3.0)
    with pytest.raises(octgpu.ConfigError):
        e.mcs(octgpu.UpdateParams.make(0.5, 0.0), torch.zeros(e.boundary_bytes, dtype=torch.uint8, device="cuda"), 2)
    with pytest.raises(octgpu.ConfigError):
        StripeEngine(cfg, 0, 5, 3)  # fewer rows than the halo a pass reads (6)


@pytest.mark.parametrize("transport", ["host", "peer-streams"])
def test_stripes_mixed_modes_lazy_streams(transport):
    """Constant-xi passes (2 MCS, streams owed lazily) followed by live passes: the halo rows'
    streams (advanced locally on the peer path) must stay exact."""
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        cfg = octgpu.LatticeConfig(2048, 200)
        grp, engines = _group(cfg, 4, 9, stream, transport)
        ref = octgpu.GpuEngine(cfg, 9)
        for pq, n in [((1.0, 0.0), 5), ((0.5, 0.25), 4), ((0.0, 0.0), 3), ((0.75, 0.0), 3)]:
            prm = octgpu.UpdateParams.make(*pq)
            grp.step(prm, n)
            ref.step(prm, n)
        for e in engines:
            e.sync()
        planes = np.concatenate([e.planes() for e in engines], axis=1)
        states = np.concatenate([e.states() for e in engines], axis=0)
        assert np.array_equal(planes, ref.planes())
        assert np.array_equal(states, ref.streams().states)
        assert grp.measure().power_sums == ref.measure().power_sums


def test_peer_wait_times_out_instead_of_hanging(monkeypatch):
    """A neighbour that stops stepping must surface as an error (bounded device wait), not a hang."""
    monkeypatch.setenv("OCTGPU_P2P_TIMEOUT_MS", "200")
    cfg = octgpu.LatticeConfig(1024, 64)
    engines = [StripeEngine(cfg, *stripe_bounds(64, 2, r), 4) for r in range(2)]
    PeerLocalTransport(engines)
    prm = octgpu.UpdateParams.make(0.5, 0.0)
    engines[0].pass_(prm, 1)  # needs the neighbours' pass 0: fine
    engines[0].pass_(prm, 1)  # needs stripe 1's pass 1, which never comes
    with pytest.raises(octgpu.CudaError, match="timed out"):
        engines[0].sync()
    for e in engines:
        e.disconnect()
