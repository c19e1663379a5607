"""Row stripes across GPUs: one stripe engine per GPU.

Partition: contiguous row blocks exactly as the reference's SweepPlan
(params.hpp:107-127; the result is partition-independent, like the
reference's worker count). Per pass of k MCS (k = 3 for constant-xi
parameters: the temporally blocked kernel, 2 for a remainder of 2; else 1),
stripe r (rows [y0, y1), at least 6):

  1. pack      rows y0..y0+5 (+ rng states) -> to_prev; rows y1-5..y1-1 (+ states) -> to_next
  2. exchange  shift-up   (to_prev -> rank r-1, from_next <- rank r+1)
               shift-down (to_next -> rank r+1, from_prev <- rank r-1)
  3. unpack    halo rows y0-5..y0-1 (from_prev) and y1..y1+5 (from_next)
  4. mcs       k fused MCS over the stripe's rows (k_mcs_deep / k_mcs_bulk)
  5. boundary  y-plane f of row y1 -> rank r+1, which completes its row y0 (finish)

The halo traffic is 11 x 4 plane-rows + one plane-row per stripe boundary
per pass (X/16 bytes per plane-row), independent of the stripe height. Measurement: every stripe reduces its own rows in a local height
gauge; the exact int128 power sums are shifted binomially by the column-0
prefix of the stripes above and summed (``combine``).

Transports: ``LocalTransport`` (all stripes in this process, e.g. several
stripes on one GPU — used to prove bit-exactness on one device) and
``DistTransport`` (one stripe per rank over torch.distributed: NCCL on GPUs,
gloo on CPU for the protocol tests) run steps 1-5 from the host.
``PeerLocalTransport`` / ``PeerDistTransport`` replace them with the
device-side exchange over peer memory (csrc/p2p.cu, csrc/stripe_link.cuh): a
multi-MCS pass between stripes on different GPUs is ONE kernel whose boundary
blocks wait on the neighbours' "passes done" counters, read their rows over
NVLink, and publish the pass; otherwise a pass is a halo pull kernel, the MCS
kernel, and one kernel that writes the boundary plane-row into the next stripe
and publishes the pass — no NCCL, no host synchronisation between passes. Peers
are mapped with CUDA IPC across processes.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import IPC_BYTES, ConfigError, OctMoments, OctPeer, OctStripeMoments, check, lib
from .engine import MeasurementRecord, _i128, _word_dtype
from .params import LatticeConfig, UpdateParams


def stripe_bounds(Y: int, parts: int, index: int) -> tuple[int, int]:
    """Row block `index` of `parts` (SweepPlan::make, params.hpp:111-126)."""
    if parts < 1:
        raise ConfigError("worker count must be >= 1")
    n = min(parts, Y)
    base, rem = divmod(Y, n)
    y = 0
    for i in range(n):
        ln = base + (1 if i >= n - rem else 0)
        if i == index:
            return y, y + ln
        y += ln
    raise ConfigError(f"stripe index {index} out of range for {n} stripes")


@dataclass
class StripeMoments:
    """Exact per-stripe statistics in the stripe-local gauge."""

    y0: int
    t: int
    n_sites: int
    sums: tuple  # (S1, S2, S3, S4)
    col_sum: int
    sy_first: int
    row_first_sum: int
    curl_count: int
    curl_first: int  # global y * X + x, or -1

    def to_array(self) -> np.ndarray:
        vals = [self.y0, self.t, self.n_sites, self.col_sum, self.sy_first, self.row_first_sum, self.curl_count,
                self.curl_first]
        for s in self.sums:
            vals += [s & 0xFFFFFFFFFFFFFFFF, (s >> 64) & 0xFFFFFFFFFFFFFFFF]
        return np.array([v & 0xFFFFFFFFFFFFFFFF for v in vals], np.uint64).view(np.int64)

    @staticmethod
    def from_array(a: np.ndarray) -> "StripeMoments":
        u = [int(v) for v in np.asarray(a, np.int64).view(np.uint64)]
        sg = lambda v: v - (1 << 64) if v >> 63 else v  # noqa: E731
        sums = tuple(_i128(u[8 + 2 * k], u[9 + 2 * k]) for k in range(4))
        return StripeMoments(u[0], u[1], u[2], sums, sg(u[3]), sg(u[4]), sg(u[5]), u[6], sg(u[7]))


def combine(parts: list[StripeMoments], X: int, Y: int) -> MeasurementRecord:
    """Global measure_heights from stripe-local sums (octgpu_stripes_combine: reconstruct_heights'
    checks in its order, slope_field.hpp:209-226, and the binomial shift of the exact int128 sums
    by the column-0 prefix of the stripes above). Host-only."""
    parts = sorted(parts, key=lambda m: m.y0)
    arr = (OctStripeMoments * len(parts))()
    mask = (1 << 64) - 1
    for a, m in zip(arr, parts):
        a.t, a.n_sites = m.t, m.n_sites
        for k in range(4):
            a.s_lo[k] = m.sums[k] & mask
            hi = (m.sums[k] >> 64) & mask
            a.s_hi[k] = hi - (1 << 64) if hi >> 63 else hi
        a.col_sum, a.sy_first, a.row_first_sum = m.col_sum, m.sy_first, m.row_first_sum
        a.curl_count = m.curl_count
        a.curl_first = m.curl_first if m.curl_count else mask
    out = OctMoments()
    check(lib().octgpu_stripes_combine(arr, len(parts), X, Y, C.byref(out)))
    sums = tuple(_i128(int(out.s_lo[k]), int(out.s_hi[k])) for k in range(4))
    return MeasurementRecord(int(out.t), out.W2, out.mean_h, out.skew, out.kurt, int(out.n_sites), sums)


class StripeEngine:
    """One row stripe [y0, y1) of an X x Y periodic lattice on one GPU."""

    def __init__(self, cfg: LatticeConfig, y0: int, y1: int, seed: int = 1, device: int = 0,
                 planes: np.ndarray | None = None, states: np.ndarray | None = None, t: int = 0, phase: int = 0):
        self._h = None
        self.cfg, self.y0, self.y1, self.device = cfg, y0, y1, device
        h = C.c_void_p()
        pp = sp = None
        if planes is not None:
            planes = np.ascontiguousarray(planes, _word_dtype(cfg.w))
            states = np.ascontiguousarray(states, np.uint64)
            pp, sp = planes.ctypes.data_as(C.c_void_p), states.ctypes.data_as(C.c_void_p)
        check(lib().octgpu_create_stripe(cfg.X, cfg.Y, cfg.w, y0, y1, t, phase, pp, sp, seed, device, C.byref(h)))
        self._h = h
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib().octgpu_stripe_sizes(h, C.byref(a), C.byref(b), C.byref(c)))
        self.to_prev_bytes, self.to_next_bytes, self.boundary_bytes = a.value, b.value, c.value

    def __del__(self, _lib=lib):  # the module global may already be gone at interpreter shutdown
        if getattr(self, "_h", None):
            _lib().octgpu_destroy(self._h)
            self._h = None

    @staticmethod
    def _p(buf) -> C.c_void_p:
        return C.c_void_p(buf.data_ptr())

    def set_stream(self, cuda_stream: int | None) -> None:
        check(lib().octgpu_set_stream(self._h, C.c_void_p(cuda_stream) if cuda_stream else None))

    def pass_plan(self, prm) -> tuple[str, float]:
        """(kernel, MCS per launch) of this stripe's passes for prm (octgpu_pass_plan)."""
        from .engine import GpuEngine
        c = prm.to_c()
        k, sw = C.c_int(), C.c_int()
        check(lib().octgpu_pass_plan(self._h, C.byref(c), C.byref(k), C.byref(sw)))
        return GpuEngine.KERNELS[k.value], sw.value / 2

    def set_rng(self, kind: str) -> None:
        """GpuEngine.set_rng for this stripe: every stripe of a group must use the same kind (the counter
        streams are keyed by the master seed and the GLOBAL row, so a striped run equals the periodic one)."""
        from .engine import GpuEngine
        if kind not in GpuEngine.RNG_KINDS:
            raise ValueError(f"rng kind must be one of {sorted(GpuEngine.RNG_KINDS)}")
        check(lib().octgpu_set_rng(self._h, GpuEngine.RNG_KINDS[kind]))

    def pack(self, to_prev, to_next) -> None:
        check(lib().octgpu_halo_pack(self._h, self._p(to_prev), self._p(to_next)))

    def unpack(self, from_prev, from_next) -> None:
        check(lib().octgpu_halo_unpack(self._h, self._p(from_prev), self._p(from_next)))

    def mcs(self, prm: UpdateParams, boundary_out, n: int = 1) -> None:
        c = prm.to_c()
        check(lib().octgpu_stripe_mcs_n(self._h, C.byref(c), n, self._p(boundary_out)))

    def max_mcs(self, prm: UpdateParams) -> int:
        """MCS one halo exchange can cover for these parameters (1, or 2 with constant xi)."""
        c = prm.to_c()
        k = int(lib().octgpu_stripe_max_mcs(self._h, C.byref(c)))
        if k < 1:
            check(1)
        return k

    def finish(self, boundary_in) -> None:
        check(lib().octgpu_stripe_finish(self._h, self._p(boundary_in)))

    # ---- device-side exchange over peer memory ----
    def peer(self) -> OctPeer:
        out = OctPeer()
        check(lib().octgpu_stripe_peer(self._h, C.byref(out)))
        return out

    def ipc_export(self) -> bytes:
        buf = C.create_string_buffer(IPC_BYTES)
        check(lib().octgpu_stripe_ipc_export(self._h, buf))
        return buf.raw

    def ipc_open(self, blob: bytes) -> OctPeer:
        out = OctPeer()
        check(lib().octgpu_stripe_ipc_open(self._h, C.create_string_buffer(blob, IPC_BYTES), C.byref(out)))
        return out

    def connect(self, prev: OctPeer, nxt: OctPeer) -> None:
        check(lib().octgpu_stripe_connect(self._h, C.byref(prev), C.byref(nxt)))

    def pass_(self, prm: UpdateParams, n: int = 1) -> None:
        c = prm.to_c()
        check(lib().octgpu_stripe_pass(self._h, C.byref(c), n))

    def pull(self) -> None:
        check(lib().octgpu_stripe_pull(self._h))

    def disconnect(self) -> None:
        check(lib().octgpu_stripe_disconnect(self._h))

    def checksum(self) -> int:
        """field_checksum of this stripe's own rows as an (y1 - y0)-row field (slope_field.hpp:232-246);
        sync the whole group first (the first row is completed by the previous stripe's push)."""
        v = C.c_uint64()
        check(lib().octgpu_field_checksum(self._h, C.byref(v)))
        return int(v.value)

    def balances(self) -> tuple[np.ndarray, np.ndarray]:
        """(row_balances of this stripe's rows, col_balances summed over them); the lattice's
        col_balances is the sum over all stripes (slope_field.hpp:177-202)."""
        rows = np.zeros(self.y1 - self.y0, np.int64)
        cols = np.zeros(self.cfg.X, np.int64)
        check(lib().octgpu_balances(self._h, rows.ctypes.data_as(C.c_void_p), cols.ctypes.data_as(C.c_void_p)))
        return rows, cols

    def measure_local(self) -> StripeMoments:
        m = OctStripeMoments()
        check(lib().octgpu_measure_stripe(self._h, C.byref(m)))
        sums = tuple(_i128(int(m.s_lo[k]), int(m.s_hi[k])) for k in range(4))
        first = int(m.curl_first) if m.curl_count else -1
        return StripeMoments(self.y0, int(m.t), int(m.n_sites), sums, int(m.col_sum), int(m.sy_first),
                             int(m.row_first_sum), int(m.curl_count), first)

    @property
    def t(self) -> int:
        return int(lib().octgpu_t(self._h))

    @property
    def launches(self) -> int:
        return int(lib().octgpu_launch_count(self._h))

    def planes(self, out: np.ndarray | None = None) -> np.ndarray:
        shape, dt = (4, self.y1 - self.y0, self.cfg.words_per_row()), _word_dtype(self.cfg.w)
        if out is None:
            out = np.zeros(shape, dt)
        elif out.shape != shape or out.dtype != dt or not out.flags.c_contiguous:
            raise ConfigError(f"planes buffer must be a C-contiguous {dt.__name__} array of shape {shape}")
        check(lib().octgpu_get_planes(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def states(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.zeros((self.y1 - self.y0, 4), np.uint64)
        elif out.shape != (self.y1 - self.y0, 4) or out.dtype != np.uint64 or not out.flags.c_contiguous:
            raise ConfigError(f"states buffer must be a C-contiguous uint64 array of shape ({self.y1 - self.y0}, 4)")
        check(lib().octgpu_get_states(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def sync(self) -> None:
        check(lib().octgpu_sync(self._h))


def _bind_current_stream(engines) -> None:
    """Host-driven transports copy halo buffers with torch (LocalTransport) or NCCL (DistTransport) on the
    current torch stream, while each stripe enqueues pack / MCS / finish on its own stream. Binding every
    GPU stripe to the current torch stream at construction orders the two; the caller keeps that stream
    current while stepping the group (set_stream() afterwards would break the ordering)."""
    import torch

    for e in engines:
        if isinstance(e, StripeEngine) and torch.cuda.is_available():
            e.set_stream(torch.cuda.current_stream(e.device).cuda_stream)


class _Buffers:
    def __init__(self, eng, alloc):
        self.tp = alloc(eng.to_prev_bytes)
        self.tn = alloc(eng.to_next_bytes)
        self.rp = alloc(eng.to_next_bytes)   # from prev = its to_next
        self.rn = alloc(eng.to_prev_bytes)   # from next = its to_prev
        self.bo = alloc(eng.boundary_bytes)
        self.bi = alloc(eng.boundary_bytes)


class LocalTransport:
    """All stripes live in this process (ring order = list order)."""

    def __init__(self, engines: list, alloc):
        self.engines = engines
        _bind_current_stream(engines)
        self.bufs = [_Buffers(e, alloc) for e in engines]

    def halos(self):
        n = len(self.engines)
        for e, b in zip(self.engines, self.bufs):
            e.pack(b.tp, b.tn)
        for r, b in enumerate(self.bufs):
            b.rp.copy_(self.bufs[(r - 1) % n].tn)
            b.rn.copy_(self.bufs[(r + 1) % n].tp)
        for e, b in zip(self.engines, self.bufs):
            e.unpack(b.rp, b.rn)

    def boundary(self):
        n = len(self.engines)
        for r, b in enumerate(self.bufs):
            b.bi.copy_(self.bufs[(r - 1) % n].bo)
        for e, b in zip(self.engines, self.bufs):
            e.finish(b.bi)

    def gather(self, parts: list[StripeMoments]) -> list[StripeMoments]:
        return parts


class DistTransport:
    """One stripe per rank of the default torch.distributed group (ring by rank)."""

    def __init__(self, engine, alloc):
        import torch.distributed as dist

        self.dist = dist
        self.engines = [engine]
        _bind_current_stream(self.engines)
        self.bufs = [_Buffers(engine, alloc)]
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        self.prev, self.next = (self.rank - 1) % self.size, (self.rank + 1) % self.size

    def _shift(self, send, to, recv, frm):
        d = self.dist
        if to == self.rank:  # world size 1
            recv.copy_(send)
            return
        ops = [d.P2POp(d.isend, send, to), d.P2POp(d.irecv, recv, frm)]
        for req in d.batch_isend_irecv(ops):
            req.wait()

    def halos(self):
        e, b = self.engines[0], self.bufs[0]
        e.pack(b.tp, b.tn)
        if self.size == 1:
            b.rn.copy_(b.tp)
            b.rp.copy_(b.tn)
        else:  # shift up and shift down in one batch (per-peer order matches sends to receives)
            d = self.dist
            ops = [d.P2POp(d.isend, b.tp, self.prev), d.P2POp(d.irecv, b.rn, self.next),
                   d.P2POp(d.isend, b.tn, self.next), d.P2POp(d.irecv, b.rp, self.prev)]
            for req in d.batch_isend_irecv(ops):
                req.wait()
        e.unpack(b.rp, b.rn)

    def boundary(self):
        e, b = self.engines[0], self.bufs[0]
        self._shift(b.bo, self.next, b.bi, self.prev)
        e.finish(b.bi)

    def gather(self, parts: list[StripeMoments]) -> list[StripeMoments]:
        import torch

        mine = torch.from_numpy(parts[0].to_array())
        dev = self.bufs[0].tp.device
        mine = mine.to(dev)
        out = [torch.empty_like(mine) for _ in range(self.size)]
        self.dist.all_gather(out, mine)
        return [StripeMoments.from_array(o.cpu().numpy()) for o in out]


class PeerLocalTransport:
    """All stripes in this process, exchanging halos device-side over peer memory."""

    peer = True

    def __init__(self, engines: list):
        self.engines = engines
        peers = [e.peer() for e in engines]
        n = len(engines)
        for r, e in enumerate(engines):
            e.connect(peers[(r - 1) % n], peers[(r + 1) % n])

    def gather(self, parts: list[StripeMoments]) -> list[StripeMoments]:
        return parts


class PeerDistTransport:
    """One stripe per rank; the ring neighbours' device memory is mapped with CUDA
    IPC (handles exchanged once over torch.distributed), then every pass runs
    device-side (csrc/p2p.cu). torch.distributed only gathers the moments."""

    peer = True

    def __init__(self, engine, device=None):
        import torch.distributed as dist

        self.dist = dist
        self.engines = [engine]
        self.rank, self.size = dist.get_rank(), dist.get_world_size()
        self.device = device
        blobs = [None] * self.size
        dist.all_gather_object(blobs, engine.ipc_export())
        prev, nxt = (self.rank - 1) % self.size, (self.rank + 1) % self.size
        if self.size == 1:
            p = q = engine.peer()
        else:
            p = engine.ipc_open(blobs[prev])
            q = p if nxt == prev else engine.ipc_open(blobs[nxt])
        engine.connect(p, q)
        dist.barrier()

    def close(self) -> None:
        """Unmap the neighbours on every rank before any rank frees its stripe."""
        self.engines[0].disconnect()
        self.dist.barrier()

    def gather(self, parts: list[StripeMoments]) -> list[StripeMoments]:
        """One fixed-size all_gather of the 16-word moment records (device tensors on NCCL, host tensors on gloo;
        no pickling: this sits inside every timed W^2 point of a multi-GPU run)."""
        import torch

        mine = torch.from_numpy(parts[0].to_array())
        if self.dist.get_backend() == "nccl":
            mine = mine.to(torch.device("cuda", torch.cuda.current_device()))
        out = torch.empty(self.size * mine.numel(), dtype=mine.dtype, device=mine.device)
        self.dist.all_gather_into_tensor(out, mine)
        host = out.cpu().numpy().reshape(self.size, -1)
        return [StripeMoments.from_array(host[r]) for r in range(self.size)]


class StripeGroup:
    """Drives stripe engines through the per-MCS protocol above."""

    def __init__(self, transport, X: int, Y: int):
        self.tr, self.X, self.Y = transport, X, Y

    def step(self, prm: UpdateParams, n: int = 1) -> None:
        kmax = self.tr.engines[0].max_mcs(prm)  # the same on every rank (depends on params and X * Ytot only)
        peer = getattr(self.tr, "peer", False)
        while n > 0:
            k = min(n, kmax)
            if peer:
                for e in self.tr.engines:
                    e.pass_(prm, k)
            else:
                self.tr.halos()
                for e, b in zip(self.tr.engines, self.tr.bufs):
                    e.mcs(prm, b.bo, k)
                self.tr.boundary()
            n -= k

    def measure(self) -> MeasurementRecord:
        # the curl check of each stripe's first row reads the row above
        if getattr(self.tr, "peer", False):
            for e in self.tr.engines:
                e.pull()
        else:
            self.tr.halos()
        parts = self.tr.gather([e.measure_local() for e in self.tr.engines])
        return combine(parts, self.X, self.Y)

    def sync(self) -> None:
        """Drain every stripe's stream (a stripe's first row is completed by its neighbour's
        boundary push, so download planes only after syncing the whole group)."""
        for e in self.tr.engines:
            e.sync()

    @property
    def t(self) -> int:
        return self.tr.engines[0].t
