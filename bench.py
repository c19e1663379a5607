#!/usr/bin/env python
"""Benchmark: site updates/ns of the bit-vectorized octahedron SCA on B200.

Workload (default, BASELINE.json configs[1]): a 2^16 x 2^16 lattice from the
flat start, KPZ p=1 q=0, one MCS per step, W^2(t) measured on the device at
the points of log_schedule(10^4, 8) that fall inside the K timed steps. The
timed steps are the LAST K MCS of the 10^4-MCS configs[1] job (the state at
t = 10^4 - K is prepared untimed; K = 10^4 runs the job whole), so a short K
measures a representative stretch rather than the W^2-dense first MCS;
--from-flat times MCS 1..K instead (c4 always does: 10 ms/MCS). Inputs: the slope
planes are 1 GiB, far larger than the 126 MB L2, so no L2 flush is needed.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c2h|c3|c4|c5] [--impl ours|reference]

Prints ONE JSON line (rank 0). --impl reference times the reference's own
multi-threaded CPU VecEngine (oracle/_ref, built from /root/reference) on
this host's cores on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(X=1 << 16, Y=1 << 16, p=1.0, q=0.0,
               workload="2^16x2^16 KPZ p=1 q=0, W^2(t) log-sampled (BASELINE configs[1])"),
    "c2h": dict(X=1 << 16, Y=1 << 16, p=0.5, q=0.0,
                workload="2^16x2^16 KPZ p=0.5 q=0 (half mode; paper's benchmark case), W^2(t) log-sampled"),
    "c3": dict(X=1 << 16, Y=1 << 16, p=0.5, q=0.5, workload="2^16x2^16 EW-like p=q=1/2 (BASELINE configs[2])"),
    "c4": dict(X=1 << 16, Y=1 << 16, p=0.98, q=0.02, window=False,  # 10 ms/MCS: no untimed 10^4-MCS prefix
               workload="2^16x2^16 arbitrary p=0.98 q=0.02 (BASELINE configs[3])"),
    "c5": dict(X=1 << 17, Y=1 << 17, p=1.0, q=0.0, workload="2^17x2^17 KPZ p=1 q=0 (BASELINE configs[4])",
               multi="strong"),
}
METRIC = "site updates/ns"
# The other BASELINE configs, timed in short windows after the headline (single GPU): MCS per window. Each
# window is the job's last K MCS like the headline (c4, 10 ms/MCS: MCS 1..K from the flat start).
CONFIG_WINDOWS = {"c2h": 50, "c3": 50, "c4": 10, "c5": 20}
CONFIG_CPU_BUDGET = 6.0  # seconds of reference CPU work per config
SCHEDULE_TMAX, SCHEDULE_PPD = 10000, 8


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clock + throttle reasons via NVML during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting",
               0x10: "sync_boost"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.stop_ev = [], set(), threading.Event()
        self.max_mhz = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.th = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self.stop_ev.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop_ev.wait(0.05)

    def __enter__(self):
        if self.nv:
            self.th.start()
        return self

    def __exit__(self, *a):
        self.stop_ev.set()
        if self.nv:
            self.th.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2], "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(s)}


def _traffic(kernel: str, config: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)[kernel][config]["dram_bytes_per_launch"]
    except Exception:
        return None


def _int_pipe(kernel: str, config: str):
    """Integer-issue evidence for the same kernel from the committed ncu capture (the arbitrary-p
    configs are ALU-pipe bound, not HBM bound): issue-active and ALU / FMA pipe utilisation in %
    of the SM's peak."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            k = json.load(f)[kernel][config]
        return {"issue_active_pct": k["issue_active_pct"], "pipe_alu_pct": k.get("pipe_alu_pct"),
                "pipe_fma_pct": k.get("pipe_fma_pct"), "dram_pct_peak": k["dram_pct_peak"],
                "source": "ncu --set full (profiles/ncu_summary.json)"}
    except Exception:
        return None


def _sync_all(engines) -> None:
    """Drain every engine's stream (a helper, so no loop variable keeps an engine - and its plane sets -
    alive after the caller drops it: the next engine then reuses the pooled memory)."""
    for eng in engines:
        eng.sync()


def timed_window(K: int, from_flat: bool, schedule: list[int]):
    """The timed K MCS are the LAST K MCS of the 10^4-MCS job (the state at t_start = 10^4 - K is prepared
    untimed), with the job's W^2 points inside that window: K = 10^4 (default) is the whole job; a short K
    measures a representative stretch instead of the W^2-dense first MCS. from_flat: MCS 1..K.
    Returns (t_start, W^2 points in the window, step targets, description)."""
    t_start = 0 if from_flat else max(0, SCHEDULE_TMAX - K)
    sched = [t for t in schedule if t_start < t <= t_start + K]
    targets = sched + ([t_start + K] if not sched or sched[-1] != t_start + K else [])
    span = (f"the {SCHEDULE_TMAX}-MCS job" if t_start + K <= SCHEDULE_TMAX
            else f"the {SCHEDULE_TMAX}-MCS job and {t_start + K - SCHEDULE_TMAX} MCS more")
    desc = (f"MCS {t_start + 1}..{t_start + K} of {span} with its {len(sched)} W^2 points; "
            + (f"state at t={t_start} prepared untimed" if t_start else "from the flat start"))
    return t_start, sched, targets, desc


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


_REF = {}


def _cpu_info() -> tuple[str, int]:
    """(CPU model of this host, usable hardware threads), taken once before the reference library loads:
    libgomp with OMP_PROC_BIND=close pins the loading thread to one CPU, which would shrink the affinity mask."""
    if "cpu" in _REF:
        return _REF["cpu"]
    model = "unknown CPU"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    _REF["cpu"] = (model, cores)
    return model, cores


def _ref_lib():
    """The reference's own VecEngine for the CPU arm: built on THIS host with -march=native from the
    reference sources shipped in baseline/_ref/proj (oracle/Makefile `native`, once per host), else the
    prebuilt oracle/_ref/libocref.so (-march=x86-64-v3). Returns (RefLib, build description)."""
    if "lib" in _REF:
        return _REF["lib"], _REF["build"]
    _cpu_info()
    os.environ.setdefault("OMP_PROC_BIND", "close")  # read by libgomp when the library loads
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import REF_SO, RefLib

    native = os.path.join(ROOT, "baseline", "_ref", "libocref_native.so")
    src = os.path.join(ROOT, "baseline", "_ref", "proj", "include", "octsca", "engine_vec.hpp")
    note = ""
    if not os.path.exists(native) and os.path.exists(src):
        import fcntl
        import subprocess

        with open(os.path.join(ROOT, "baseline", "_ref", ".build.lock"), "w") as lk:
            fcntl.flock(lk, fcntl.LOCK_EX)  # the driver may start both arms back to back
            if not os.path.exists(native):
                r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "native"],
                                   capture_output=True, text=True, timeout=600)
                if r.returncode:
                    note = f" (native build failed: {r.stderr.strip().splitlines()[-1:] or r.returncode})"
    lib, build = None, None
    if os.path.exists(native):
        try:
            lib, build = RefLib(native), "reference sources compiled on this host: g++ -std=c++20 -O3 -march=native -fopenmp"
        except OSError as ex:
            note = f" (native library failed to load: {ex})"
    if lib is None:
        lib, build = RefLib(REF_SO), "prebuilt oracle/_ref/libocref.so: g++ -std=c++20 -O3 -march=x86-64-v3 -fopenmp" + note
    _REF["lib"], _REF["build"] = lib, build
    return lib, build


def cpu_reference_run(cfg: dict, steps: int, warmup: int, budget_s: float):
    """Time the reference's VecEngine<uint64_t> (engine_vec.hpp:184-213) on this host's cores: `warmup`
    (at most 1) untimed MCS, then MCS until `steps` or the time budget (at least one).
    Returns (updates/ns, threads, MCS timed, seconds, description)."""
    lib, build = _ref_lib()  # puts oracle/ on sys.path
    from oracle import RefEngine

    model, cores = _cpu_info()
    X, Y = cfg["X"], cfg["Y"]
    eng = RefEngine(lib, X, Y, 1, workers=cores)
    for _ in range(max(0, min(warmup, 1))):
        eng.step(cfg["p"], cfg["q"], 1)
    done, t0 = 0, time.perf_counter()
    while done < max(1, steps):
        eng.step(cfg["p"], cfg["q"], 1)
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    desc = (f"{done} MCS of {X}x{Y} p={cfg['p']} q={cfg['q']} after {min(warmup, 1)} warm-up MCS, steps only "
            f"(no W2), {el:.1f} s; VecEngine<uint64_t> workers={cores} OMP_PROC_BIND=close on {model}; {build}")
    return X * Y * done / (el * 1e9), cores, done, el, desc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=SCHEDULE_TMAX)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of CPU reference work")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the short windows of the other BASELINE configs (c2h, c3, c4, c5) in the c2 line")
    ap.add_argument("--from-flat", action="store_true", help="time MCS 1..K instead of the job's last K MCS")
    ap.add_argument("--rng", default="xoshiro", choices=["xoshiro", "counter"],
                    help="xi source: the reference's xoshiro streams, or the opt-in counter-based mode "
                         "(not bit-compatible with the reference; single GPU)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    ws, rank, local = _dist()
    K, W = args.steps, max(3, args.warmup)
    # N > 1: c5 is one fixed 2^17 x 2^17 lattice striped over the GPUs (strong scaling, BASELINE configs[4]);
    # the 2^16 x 2^16 configs keep 2^16 x 2^16 sites per GPU: an X x (N * 2^16) lattice in N row stripes (weak)
    scaling = cfg.get("multi", "weak")
    if ws > 1 and scaling == "weak":
        cfg["Y"] = cfg["Y"] * ws
        cfg["workload"] += f"; {ws} GPUs: {cfg['X']}x{cfg['Y']} lattice, one 2^16-row stripe per GPU"

    if args.rng != "xoshiro" and args.impl == "reference":
        raise SystemExit("--rng counter: our implementation only (the reference has no counter rng)")
    config_key = {"workload": cfg["workload"], "X": cfg["X"], "Y": cfg["Y"], "p": cfg["p"], "q": cfg["q"],
                  "w": 64, "seed": 1, "schedule": f"log_schedule({SCHEDULE_TMAX},{SCHEDULE_PPD}) within steps",
                  "l2": "planes (>=1 GiB) exceed L2 (126 MB); no flush needed", "parallelism": f"row stripes x{ws}" if ws > 1 else "single GPU"}
    if args.rng != "xoshiro":
        config_key["rng"] = "counter (opt-in SplitMix64 streams, octgpu_set_rng; not the reference's generator)"

    if args.impl == "reference":
        if rank != 0:
            return
        v, cores, done, el, sample = cpu_reference_run(cfg, K, W, args.cpu_budget)
        line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "updates/ns",
                "n_gpus": ws, "steps": done, "warmup": min(W, 1), "ms_per_step": el * 1e3 / done,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (flat start, seed 1)", "config": config_key,
                "cpu_baseline": {"value": v, "unit": "updates/ns", "cores": cores, "kind": "reference",
                                 "sample": sample},
                "e2e": {"value": v, "unit": "updates/ns", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        if ws == 1 and args.config == "c2" and not args.no_configs:
            line["configs"] = {}
            for name in CONFIG_WINDOWS:
                c = CONFIGS[name]
                cv, cc, cd, cel, cs = cpu_reference_run(c, 1000, 1, CONFIG_CPU_BUDGET)
                line["configs"][name] = {"workload": c["workload"], "value": cv, "unit": "updates/ns",
                                         "ms_per_mcs": cel * 1e3 / cd, "cores": cc, "sample": cs}
        print(json.dumps(line))
        return

    import numpy as np
    import torch

    import paper_1606_00310_b200 as octgpu

    # OCTGPU_BENCH_ONE_GPU=1 (protocol check only, timings meaningless): every rank on cuda:0, gloo
    one_gpu = os.environ.get("OCTGPU_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            # NCCL's communicator lines (ranks, devices, NVLink / NVLS paths) on stderr, for the run record
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
            torch.distributed.barrier()  # create the communicator now (eagerly, so it is logged up front)
    stream = torch.cuda.Stream(dev)  # a real (non-default) stream shared by the engine and the timing events
    torch.cuda.set_stream(stream)

    X, Y = cfg["X"], cfg["Y"]
    lat = octgpu.LatticeConfig(X, Y, 64)
    prm = octgpu.UpdateParams.make(cfg["p"], cfg["q"])
    t_start, sched, targets, config_key["window"] = timed_window(
        K, args.from_flat or not cfg.get("window", True), octgpu.log_schedule(SCHEDULE_TMAX, SCHEDULE_PPD))

    def barrier():
        if ws > 1:
            torch.distributed.barrier()

    def make(planes=None, states=None, t=0):
        """The job's engine: one GpuEngine, or this rank's row stripe (peer-memory / NCCL halo exchange)."""
        if ws == 1:
            if planes is None:
                eng = octgpu.GpuEngine(lat, 1, device=local)
            else:
                eng = octgpu.GpuEngine(octgpu.SlopeField(lat, planes, t, 0), octgpu.RngStreamSet(1, states),
                                       device=local)
            eng.set_stream(stream.cuda_stream)
            if args.rng != "xoshiro":
                eng.set_rng(args.rng)
            return eng, [eng]
        from paper_1606_00310_b200.stripes import (DistTransport, PeerDistTransport, StripeEngine, StripeGroup,
                                                   stripe_bounds)
        y0, y1 = stripe_bounds(Y, ws, rank)
        e = StripeEngine(lat, y0, y1, 1, device=local, planes=planes, states=states, t=t)  # this rank's rows
        e.set_stream(stream.cuda_stream)
        if args.rng != "xoshiro":
            e.set_rng(args.rng)
        alloc = lambda nb: torch.zeros(nb, dtype=torch.uint8, device=dev)  # noqa: E731
        return StripeGroup(_transport(e, alloc, PeerDistTransport, DistTransport), X, Y), [e]

    transport_used = []

    def _close(job):
        tr = getattr(job, "tr", None)
        if tr is not None and hasattr(tr, "close"):
            tr.close()

    def _transport(e, alloc, peer_cls, nccl_cls):
        """Device-side peer-memory halo exchange (csrc/p2p.cu) unless OCTGPU_TRANSPORT=nccl or any rank
        cannot map its neighbours (then every rank falls back to the NCCL host protocol)."""
        ok, tr = 0, None
        if os.environ.get("OCTGPU_TRANSPORT", "p2p") == "p2p":
            try:
                tr, ok = peer_cls(e), 1
            except Exception as ex:  # noqa: BLE001 - reported in the JSON line
                transport_used.append(f"p2p unavailable: {ex}")
        flag = torch.tensor([ok], device=dev)
        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
        if int(flag[0]) == 1:
            transport_used.append("p2p (device-side halo exchange over peer memory)")
            return tr
        transport_used.append("nccl (host-driven isend/irecv)")
        return nccl_cls(e, alloc)

    # ---- warm-up (separate engine; the timed run starts from the flat state) ----
    job, engs = make()
    job.step(prm, W)
    job.measure()
    torch.cuda.synchronize()
    _close(job)
    del job, engs
    torch.cuda.synchronize()

    def timed(job, engs, prm_, t0_, sched_, targets_, clk_device=None):
        """The K timed MCS (targets_) of a prepared job: CUDA events on the engines' stream around the whole
        window and around each step() segment, W^2 measured at the schedule points inside the window.
        Returns (window ms, step ms, records, launches, clocks summary), max over ranks."""
        seg_events, records = [], []
        launches0 = sum(e.launches for e in engs)
        barrier()
        torch.cuda.synchronize()
        clk = ClockSampler(clk_device) if clk_device is not None else None
        if clk:
            clk.__enter__()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        t = t0_
        for target in targets_:
            if target > t:
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record(stream)
                job.step(prm_, target - t)
                b.record(stream)
                seg_events.append((a, b))
                t = target
            if target in sched_:
                records.append(job.measure())
        ev1.record(stream)
        torch.cuda.synchronize()
        if clk:
            clk.__exit__(None, None, None)
        barrier()
        ms_ = ev0.elapsed_time(ev1)
        step_ms_ = sum(a.elapsed_time(b) for a, b in seg_events)
        launches_ = sum(e.launches for e in engs) - launches0
        if ws > 1:
            tt = torch.tensor([ms_, step_ms_], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            ms_, step_ms_ = float(tt[0]), float(tt[1])
            lt = torch.tensor([launches_], device=dev)
            torch.distributed.all_reduce(lt)
            launches_ = int(lt[0])
        return ms_, step_ms_, records, launches_, (clk.summary() if clk else None)

    # ---- timed region, device-resident ----
    job, engs = make()
    if t_start:
        job.step(prm, t_start)  # untimed: the job's state at the start of the timed window
        _sync_all(engs)
    torch.cuda.synchronize()
    ms, step_ms, records, launches, clocks = timed(job, engs, prm, t_start, sched, targets, clk_device=local)
    kname, mcs_per_launch = engs[0].pass_plan(prm)  # the engine's own dispatch (octgpu_pass_plan)
    value = X * Y * K / (ms * 1e6)
    kernel_ms = step_ms / K  # per MCS, all launches of the step calls
    peak, peak_src = _peaks()
    # paper identity: 1 byte of slope traffic per site update, per GPU, per launch
    alg_bytes = int(X * Y // ws * mcs_per_launch)
    launch_ms = kernel_ms * mcs_per_launch
    achieved = alg_bytes / (launch_ms * 1e-3) / 1e9
    final_checksum = engs[0].checksum() if ws == 1 else None
    # Correctness digest of the timed job (every N): the exact global power sums S_k = sum h^k at the
    # window's last W^2 point and each stripe's field_checksum (its own rows as a field; N = 1: the
    # lattice's), with the exactly known expected values for p = 1 (below: `expected`, `verified`).
    job.sync()
    rec = records[-1] if records else job.measure()
    mine = final_checksum if final_checksum is not None else engs[0].checksum()
    allc = [hex(mine)]
    if ws > 1:
        allc = [None] * ws
        torch.distributed.all_gather_object(allc, hex(mine))
    digest = {"t": rec.t, "power_sums": [str(v) for v in rec.power_sums], "W2": rec.W2, "mean_h": rec.mean_h,
              "stripe_checksums": allc}
    _close(job)
    del job, engs
    if cfg["p"] == 1.0 and cfg["q"] == 0.0 and Y % ws == 0:
        # p = 1 from the flat start is flat again after every MCS: the expected state is known
        # exactly -- every GPU's rows are a flat X x Y/N field at the same t (its checksum, untimed) and the
        # lattice's sums are the flat ones (heights (x + y) mod 2: S_k = the sites at height 1 = X Y / 2, every k)
        rows = Y // ws
        flat_planes = np.zeros((4, rows, X // 128), np.uint64)  # new_flat (slope_field.hpp:110-118)
        flat_planes[1] = flat_planes[3] = np.iinfo(np.uint64).max
        flat = octgpu.GpuEngine(octgpu.SlopeField(octgpu.LatticeConfig(X, rows, 64), flat_planes, t_start + K, 0),
                                octgpu.RngStreamSet.derive(1, rows), device=local)
        exp_sum = hex(flat.checksum())
        del flat, flat_planes
        exp_ps = [str(X * Y // 2)] * 4
        digest["expected"] = {"power_sums": exp_ps, "stripe_checksum": exp_sum,
                              "rule": "p=1 from the flat start: flat after every MCS"}
        digest["verified"] = digest["power_sums"] == exp_ps and all(c == exp_sum for c in digest["stripe_checksums"])

    # ---- e2e through the C-ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        # this rank's input (the whole lattice, or its row stripe) in pinned host memory, and pinned
        # result buffers, prepared before the timed region
        if ws == 1:
            r0, r1 = 0, Y
        else:
            from paper_1606_00310_b200.stripes import stripe_bounds
            r0, r1 = stripe_bounds(Y, ws, rank)
        if t_start == 0:
            flat = np.zeros((4, r1 - r0, X // 128), np.uint64)  # new_flat (slope_field.hpp:110-118): rows do
            flat[1] = flat[3] = np.iinfo(np.uint64).max         # not depend on y: any row range is a flat stripe
            states0 = octgpu.RngStreamSet.derive(1, r1).states[r0:r1]
        else:  # the state at t_start, downloaded untimed
            prep, pengs = make()
            prep.step(prm, t_start)
            _sync_all(pengs)
            flat = pengs[0].planes()
            states0 = pengs[0].states() if ws > 1 else pengs[0].streams().states
            _close(prep)
            del prep, pengs
        host_planes = torch.from_numpy(np.ascontiguousarray(flat).view(np.int64)).pin_memory()
        host_states = torch.from_numpy(np.ascontiguousarray(states0).view(np.int64)).pin_memory()
        import ctypes as C
        pin_planes = torch.empty(host_planes.shape, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        pin_states = torch.empty(host_states.shape, dtype=torch.int64).pin_memory().numpy().view(np.uint64)
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hp = host_planes.numpy().view(np.uint64)
        hs = host_states.numpy().view(np.uint64)
        job, engs = make(hp, hs, t_start)
        engs[0].sync()
        t_create = time.perf_counter() - t0
        t = t_start
        n_meas = 0
        for target in targets:
            if target > t:
                job.step(prm, target - t)
                t = target
            if target in sched:
                job.measure()
                n_meas += 1
        engs[0].sync()
        t_run = time.perf_counter() - t0 - t_create
        out_planes = engs[0].planes(out=pin_planes)
        out_states = (engs[0].states(out=pin_states) if ws > 1 else engs[0].streams(out=pin_states).states)
        el = time.perf_counter() - t0
        _close(job)
        del job, engs
        if ws > 1:
            tt = torch.tensor([el], device=dev)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            el = float(tt[0])
        e2e = {"value": X * Y * K / (el * 1e9), "unit": "updates/ns",
               "h2d_bytes_per_step": ws * (hp.nbytes + hs.nbytes) / K,
               "d2h_bytes_per_step": (ws * (out_planes.nbytes + out_states.nbytes)
                                      + n_meas * C.sizeof(octgpu._lib.OctMoments)) / K,
               "wall_s": el, "create_s": t_create, "run_s": t_run, "d2h_s": el - t_create - t_run,
               "note": "engine(s) created from pinned host planes+states (each rank its stripe), K MCS + "
                       "measurements, planes/states D2H into pinned buffers; max over ranks"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        try:
            v, cores, done, el, sample = cpu_reference_run(cfg, 1000, 1, args.cpu_budget)
            cpu = {"value": v, "unit": "updates/ns", "cores": cores, "kind": "reference", "sample": sample}
        except Exception as ex:  # reported, never fatal
            cpu = {"value": None, "unit": "updates/ns", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    def dram(kn: str, cname: str, lms: float, sites: int | None = None):
        """ncu DRAM bytes per launch (profiles/ncu_summary.json, captured on one GPU on the config's whole lattice)
        over this run's event time per launch; `sites` = this GPU's sites when it holds a stripe (the traffic
        scales with the rows a launch processes: strong-scaled c5 stripes are 1/N of the profiled lattice)."""
        tr = _traffic(kn, cname)
        if not tr:
            return None, None, tr
        if sites is not None:
            tr = tr * sites / (CONFIGS[cname]["X"] * CONFIGS[cname]["Y"])
        gbs = tr / (lms * 1e-3) / 1e9
        return gbs, gbs / peak, tr

    # ---- the other BASELINE configs in short windows (single GPU, the c2 line only) ----
    configs = None
    if ws == 1 and args.config == "c2" and args.rng == "xoshiro" and not args.no_configs:
        configs = {}
        sched_all = octgpu.log_schedule(SCHEDULE_TMAX, SCHEDULE_PPD)
        for name, Kc in CONFIG_WINDOWS.items():
            c = CONFIGS[name]
            latc = octgpu.LatticeConfig(c["X"], c["Y"], 64)
            prmc = octgpu.UpdateParams.make(c["p"], c["q"])
            t0c, schedc, targetsc, windowc = timed_window(Kc, not c.get("window", True), sched_all)
            eng = octgpu.GpuEngine(latc, 1, device=local)
            eng.set_stream(stream.cuda_stream)
            eng.step(prmc, 2)  # warm-up of this config's kernels (plans, tensor maps), then the window's start
            eng.sync()
            eng = None
            eng = octgpu.GpuEngine(latc, 1, device=local)
            eng.set_stream(stream.cuda_stream)
            if t0c:
                eng.step(prmc, t0c)
                eng.sync()
            msc, stepc, recc, lc, clkc = timed(eng, [eng], prmc, t0c, schedc, targetsc, clk_device=local)
            kc, mplc = eng.pass_plan(prmc)
            kmsc = stepc / Kc
            lmsc = kmsc * mplc
            gbs, dfrac, trc = dram(kc, name, lmsc)
            endrec = recc[-1] if recc and recc[-1].t == t0c + Kc else eng.measure()  # W^2 at the window's end
            entry = {"workload": c["workload"], "value": c["X"] * c["Y"] * Kc / (msc * 1e6), "unit": "updates/ns",
                     "steps": Kc, "window": windowc, "ms_per_step": msc / Kc, "ms_per_mcs": kmsc,
                     "kernel": f"{kc} ({mplc} MCS per launch)", "launch_ms": lmsc,
                     "roofline_frac": c["X"] * c["Y"] * mplc / (lmsc * 1e-3) / 1e9 / peak,
                     "dram_gbs": gbs, "dram_frac": dfrac, "dram_bytes_per_launch": trc,
                     "int_pipe": _int_pipe(kc, name) if name == "c4" else None,
                     "gpu_launches": lc, "clocks": clkc, "measurements": len(recc),
                     "final_checksum": hex(eng.checksum()), "t_end": eng.t, "W2": endrec.W2,
                     "power_sums": [str(v) for v in endrec.power_sums]}
            eng = None
            if rank == 0 and not args.no_cpu_baseline:
                try:
                    cv, cc, cd, cel, cs = cpu_reference_run(c, 1000, 1, CONFIG_CPU_BUDGET)
                    entry["cpu_baseline"] = {"value": cv, "unit": "updates/ns", "cores": cc, "kind": "reference",
                                             "sample": cs}
                    entry["vs_cpu"] = entry["value"] / cv
                except Exception as ex:  # reported, never fatal
                    entry["cpu_baseline"] = {"value": None, "sample": f"unavailable: {ex}"}
            configs[name] = entry

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "updates/ns", "n_gpus": ws, "steps": K, "warmup": W,
            "ms_per_step": ms / K, "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
            "dtype": "u64", "data": "synthetic (flat start h=(x+y) mod 2, seed 1)", "config": config_key,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": dram(kname, args.config, launch_ms, X * Y // ws)[2],
                         "kernel": f"{kname} ({mcs_per_launch} MCS per launch)",
                         "alg_bytes_per_launch": alg_bytes, "launch_ms": launch_ms, "kernel_ms": kernel_ms,
                         "peak_source": peak_src, "dram_gbs": dram(kname, args.config, launch_ms, X * Y // ws)[0],
                         "dram_frac": dram(kname, args.config, launch_ms, X * Y // ws)[1],
                         "dram_per_gpu": "traffic and dram_frac are per GPU (its stripe's share of the profiled "
                                         "launch) when n_gpus > 1",
                         "note": "alg bytes = 1 B/site-update (2 slope bits x 2 reads + 2 writes per MCS); the fused "
                                 "kernels move ~0.5 B (k_mcs_bulk) / ~0.25 or ~0.17 B (k_mcs_deep, 2 or 3 MCS) of DRAM traffic per update, "
                                 "so frac exceeds 1; traffic = ncu dram bytes per launch (profiles/ncu_summary.json)"},
            "int_pipe": _int_pipe(kname, args.config),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "digest": digest,
            "transport": transport_used[-1] if transport_used else None,
            "measurements": len(records),
            "W2_last": records[-1].W2 if records else None,
            "final_checksum": hex(final_checksum) if final_checksum is not None else None,
            "configs": configs,
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
