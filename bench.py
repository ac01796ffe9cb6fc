#!/usr/bin/env python
"""Benchmark: aggregate-analysis trials/sec on the C2 workload (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3|c4] [--scaling weak|strong] [--pipeline] [--packed-ids]

--workload c3 (the 16-layer portfolio over 1M trials split across the GPUs,
allgather_portfolio between ranks) and c4 / --scaling strong (10M trials
split across the GPUs) are the other BASELINE.json configs; the default c2
line is the headline.

Workload (per GPU): 1M trials x 1000 events, one layer of
15 ELTs over a 2M-event catalog, Cat XL + Aggregate XL terms
LayerTerms(500, 10000, 140000, 66000).  ELTs come from the reference
generator restatement (seed 2066); the YET comes from `synth.bulk_yet`
(fast Philox blocks; uniform ids like the reference generator).  A step is
one pass of the hot path: K2 over this GPU's trials -> (N > 1: NCCL
all-gather of the YLT slices) -> K3 PML/TVaR at rp {10, 50, 100, 250}.

`value` times steps with inputs resident in HBM (CUDA events on the launch
stream, max over ranks); `e2e` times the same pass through the public host
API (price_layer + order_stats on pinned host buffers: H2D of the ids and
offsets, K2, D2H of the YLT, K3).  Weak scaling: N GPUs process N x 1M trials.
The 4 GB id stream per GPU is larger than L2, so no L2 flush is needed
between steps; the hot-set records stay L2-resident by design.

`--impl reference` times the reference's own CPU kernel (oracle/_ref, the
compiled _kernel.pyx; the C port when _ref is absent) on this host's cores
through the reference's thread-pool driver, on a bounded trial sample.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CATALOG = 2_000_000
EVENTS = 1000
TRIALS_PER_GPU = 1_000_000
N_ELTS = 15
TERMS = (500.0, 10_000.0, 140_000.0, 66_000.0)
RPS = [10.0, 50.0, 100.0, 250.0]
E2E_ROUNDS = 3
SEED = 2066
METRIC = "aggregate-analysis trials/sec, 1M×1000-event YET, 1/2/4/8 B200; % HBM BW"
WORKLOAD = "C2: 1M trials x 1000 events/trial per GPU, 1 layer x 15 ELTs, catalog 2M, Cat XL + Agg XL"
WORKLOAD_C3 = "C3: 1M trials x 1000 events/trial split over the GPUs, 16-layer portfolio (32-ELT pool, PO/Agg XL)"
WORKLOAD_C4 = "C4: 10M trials x 1000 events/trial split over the GPUs (strong scaling), 1 layer x 15 ELTs"


def bytes_per_trial(events: int = EVENTS, elts: int = N_ELTS) -> int:
    """4 B per id + 4 B per (event, ELT) lookup + 8 B offset + 4 B YLT."""
    return 12 + 4 * events * (1 + elts)


def host_descriptor() -> dict:
    """Logical/physical core counts and CPU model (reference bench.py:79-96)."""
    d = {"logical_cores": os.cpu_count(), "affinity_cores": host_cores(), "physical_cores": None, "cpu": None}
    try:
        import psutil

        d["physical_cores"] = psutil.cpu_count(logical=False)
    except Exception:
        pass
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    d["cpu"] = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return d


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _peaks() -> tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(kernel: str, key: str = "dram_bytes_per_launch") -> float | None:
    """Per-launch figure of K2 from the committed ncu capture of `kernel`, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "k2_traffic.json")) as f:
            d = json.load(f)
        return float(d[key]) if d.get("kernel", "k2_hotset") == kernel and d.get(key) is not None else None
    except Exception:
        return None


# Scattered-sector throughput of one B200 measured alone (K2-R):
# random 16-byte loads from an L2-resident table, scripts/micro/gather_rate.cu
SECTOR_PEAK_G_PER_S = 186.0


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.reasons |= {n for b, n in self.REASONS.items() if mask & b and b != 0x1}
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self._nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self._nv is not None:
            self._stop.set()
            self._t.join()

    def summary(self) -> dict:
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


class GpuLocalCpus:
    """Temporarily pin this thread to the CPUs NVML reports as local to the
    GPU, so pinned host buffers are first-touched on the GPU's NUMA node."""

    def __init__(self, index: int):
        self.index = index
        self.saved = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
            cpus = {w * 64 + b for w, word in enumerate(words) for b in range(64) if word >> b & 1}
            cpus &= os.sched_getaffinity(0)
            if cpus:
                self.saved = os.sched_getaffinity(0)
                os.sched_setaffinity(0, cpus)
        except Exception:
            self.saved = None
        return self

    def __exit__(self, *exc):
        if self.saved:
            os.sched_setaffinity(0, self.saved)


# ------------------------------------------------------------------ data --

def make_layer():
    from paper_1308_2066_b200.portfolio import Layer, LayerTerms
    from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt

    spec = GeneratorSpec(seed=SEED, catalog_size=CATALOG, elt_count=N_ELTS,
                         elt_size_range=(10_000, 30_000), loss_scale=1000.0)
    elts = tuple(generate_elt(spec, i) for i in range(N_ELTS))
    return Layer("c2", elts, LayerTerms(*TERMS))


def make_yet(first: int, last: int, threads: int):
    from paper_1308_2066_b200.synth import bulk_yet

    return bulk_yet(SEED, CATALOG, first, last, EVENTS, threads=threads)


# ------------------------------------------------------- reference (CPU) --

def cpu_reference(layer, yet, sample_trials: int, threads: int, steps: int = 1, warmup: int = 0) -> dict:
    """The reference CPU kernel on this host: oracle/_ref (compiled
    _kernel.pyx) when built, else the C port; the reference's threaded driver."""
    import oracle

    kind = "reference" if oracle.ref_kernel() is not None else "port"
    stacked = oracle.dense_tables(layer.elts, CATALOG)
    fin = [np.array([getattr(e.terms, f) for e in layer.elts], dtype=np.float64)
           for f in ("exchange_rate", "event_retention", "event_limit", "share")]
    sub_off = np.ascontiguousarray(yet.offsets[: sample_trials + 1])
    ids = np.ascontiguousarray(yet.event_ids[: int(sub_off[-1])])
    times = []
    for i in range(warmup + steps):
        t0 = time.perf_counter()
        oracle.run_layer_cpu(ids, sub_off, stacked, fin, TERMS, workers=threads, kernel=kind)
        dt = time.perf_counter() - t0
        if i >= warmup:
            times.append(dt)
    best = min(times)  # reference bench convention: min of rounds (bench.py:113-140)
    return {"value": sample_trials / best, "unit": "trials/s", "cores": threads, "kind": kind,
            "sample": f"first {sample_trials} trials of the same YET/ELTs/terms, "
                      f"{'oracle/_ref (compiled reference _kernel.pyx)' if kind == 'reference' else 'C port'}, "
                      f"{threads} threads via the reference _run_layer batching, min of {len(times)} rounds",
            "seconds": best}


def calibrate_sample(layer, threads: int, seconds: float) -> int:
    """Trials the CPU reference processes in about `seconds` on this host."""
    probe = max(2_000, 200 * threads)
    yet = make_yet(0, probe, threads)
    rate = cpu_reference(layer, yet, probe, threads)["value"]
    return int(min(TRIALS_PER_GPU, max(2_000, rate * seconds)))


def run_reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    layer = make_layer()
    threads = host_cores()
    # every round is a bounded sample; the whole run targets ~90 s of CPU time
    sample = args.cpu_sample or calibrate_sample(layer, threads, 90.0 / (args.steps + args.warmup))
    yet = make_yet(0, sample, threads)
    res = cpu_reference(layer, yet, sample, threads, steps=args.steps, warmup=args.warmup)
    full = None
    if not args.cpu_sample and not args.no_full_pass:
        # one pass over the whole C2 workload (1M trials) to pin the sampled
        # rate: the rate is linear in trials
        del yet
        yet_full = make_yet(0, TRIALS_PER_GPU, threads)
        f = cpu_reference(layer, yet_full, TRIALS_PER_GPU, threads, steps=1)
        full = {"trials": TRIALS_PER_GPU, "seconds": f["seconds"], "trials_per_s": f["value"],
                "sampled_over_full": res["value"] / f["value"],
                "note": "one pass of the full 1M-trial C2 workload after the sampled steps, same kernel and threads"}
        del yet_full
    line = {
        "metric": METRIC, "value": res["value"], "unit": "trials/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["seconds"] * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "sample_trials": sample, "events_per_trial": EVENTS,
                   "elts": N_ELTS, "catalog": CATALOG, "parallelism": f"{threads} host threads"},
        "cpu_baseline": dict({k: res[k] for k in ("value", "unit", "cores", "kind", "sample")}, host=host_descriptor()),
        "e2e": {"value": res["value"], "unit": "trials/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "same_config": False,
        "same_config_note": "each step is a bounded sample of the C2 YET (first `sample_trials` trials); "
                            "`full_pass` times the whole 1M-trial workload once",
    }
    if full is not None:
        line["full_pass"] = full
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- our arm --

def c3_portfolio(seed: int = SEED):
    """C3's portfolio: 16 layers over a 32-ELT pool, layer i even
    Per-Occurrence XL (occR_i, occL_i, 0, inf), odd Aggregate XL (0, inf,
    aggR_i, aggL_i), terms from the reference generator restatement."""
    import math

    from paper_1308_2066_b200.portfolio import Layer, LayerTerms
    from paper_1308_2066_b200.synth import GeneratorSpec, generate_elt, generate_layer

    spec = GeneratorSpec(seed=seed, catalog_size=CATALOG, elt_count=32, elt_size_range=(10_000, 30_000),
                         layer_count=16, elts_per_layer=15)
    pool = [generate_elt(spec, i) for i in range(32)]
    layers = []
    for i in range(16):
        g = generate_layer(spec, i, pool)
        t = g.terms
        terms = LayerTerms(t.occ_retention, t.occ_limit, 0.0, math.inf) if i % 2 == 0 else \
            LayerTerms(0.0, math.inf, t.agg_retention, t.agg_limit)
        layers.append(Layer(g.id, g.elts, terms))
    return layers


def c3_fused(dyet, stream, reps: int = 5) -> dict:
    """C3's portfolio shape on this GPU's resident ids: one fused K2 pass for
    16 layers (K2-L), CUDA events on the launch stream (a side metric of the
    C2 line; `--workload c3` is the multi-GPU C3 bench)."""
    import torch

    from paper_1308_2066_b200.direct_access import TableSet
    from paper_1308_2066_b200.engine import layer_pool, simulate_layers_device

    layers = c3_portfolio()
    pe, masks = layer_pool(layers)
    ptset = TableSet.from_elts(pe, CATALOG)
    lterms = [lay.terms for lay in layers]
    n = dyet.trial_count
    out = torch.empty((16, n), dtype=torch.float64, device=dyet.device)
    peak, _ = _peaks()
    res = {}
    for pre in (False, True):
        with torch.cuda.stream(stream):
            for _ in range(2):
                simulate_layers_device(dyet, ptset, masks, lterms, out=out, precombine=pre, check=False)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            ev[0].record(stream)
            for _ in range(reps):
                simulate_layers_device(dyet, ptset, masks, lterms, out=out, precombine=pre, check=False)
            ev[1].record(stream)
        torch.cuda.synchronize(dyet.device)
        ms = ev[0].elapsed_time(ev[1]) / reps
        hbm = n * (compulsory_bytes_per_trial() + 8 * 15)  # ids + offset once, 16 float64 YLT rows
        res["precombined" if pre else "exact"] = {
            "kernel_ms": ms, "portfolio_trials_per_s": n / (ms / 1e3), "layer_trials_per_s": 16 * n / (ms / 1e3),
            "hbm_bytes_per_launch": hbm, "achieved_gbs": hbm / (ms / 1e3) / 1e9,
            "frac": hbm / (ms / 1e3) / 1e9 / peak}
    res.update({"layers": 16, "pool_elts": 32, "trials": n,
                "note": "C3 shape, one pass over the ids for 16 layers: `exact` evaluates every (event, layer) "
                        "in K2 (k2_layers), `precombined` reads a per-event table of the 16 occurrence values "
                        "built once by K1-L (k2_layers_pre); both bitwise equal to 16 single-layer K2 runs "
                        "(tests); frac on the bytes that cross HBM (ids + offsets + 16 YLT rows)"})
    return res


def packed_side(dyet, plan, terms, d_ref, stream, n: int, k2_ms: float, rest_ms: float) -> dict | None:
    """K2 of the headline step over the packed resident ids (ARE_PACKED_IDS=1
    layout, built here beside the uint32 ids and freed after): kernel time,
    the step rate it implies (same exchange + K3), and frac on the bytes that
    then cross HBM.  Its YLT must equal the headline's bit for bit."""
    import torch

    old = os.environ.get("ARE_PACKED_IDS")
    os.environ["ARE_PACKED_IDS"] = "1"
    try:
        dyet._pack_ids()
    finally:
        if old is None:
            os.environ.pop("ARE_PACKED_IDS")
        else:
            os.environ["ARE_PACKED_IDS"] = old
    if dyet.d_packed is None:
        return None
    try:
        out = torch.empty_like(d_ref)
        for _ in range(3):
            dyet.simulate_device(plan, terms, out=out, stream=stream, check=False)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        reps = 20
        for _ in range(reps):
            dyet.simulate_device(plan, terms, out=out, stream=stream, check=False)
        ev[1].record(stream)
        torch.cuda.synchronize(dyet.device)
        ms = ev[0].elapsed_time(ev[1]) / reps
        equal = bool(torch.equal(out.view(torch.int64), d_ref.view(torch.int64)))
        hbm = int(dyet.d_packed.numel()) * 8 + 16 * n
        peak, _ = _peaks()
        return {"kernel_ms": ms, "uint32_kernel_ms": k2_ms, "step_trials_per_s": n / ((ms + rest_ms) / 1e3),
                "bytes_per_launch": hbm, "achieved_gbs": hbm / (ms / 1e3) / 1e9,
                "frac": hbm / (ms / 1e3) / 1e9 / peak, "ylt_bitwise_equal_headline": equal,
                "note": "ARE_PACKED_IDS=1: the relay kernel streams three 21-bit ids per 64-bit word "
                        "(are_yet_pack_device) -- 2/3 of the id bytes, faster K2, lower frac (fewer bytes); "
                        "opt-in because it keeps a second id copy in HBM (DESIGN.md section 4)"}
    finally:
        dyet.d_packed = None


def compulsory_bytes_per_trial(events: int = EVENTS) -> int:
    """Bytes that must cross HBM per trial: its ids, its offset, its float64 YLT slot."""
    return 4 * events + 8 + 8


def _sector_roofline(kernel: str, kernel_ms: float, trials: int) -> dict | None:
    """K2's binding bound: every id row and every record gather is an L2
    sector read through the SM's memory path (ids + records, ncu
    lts__t_sectors_srcunit_tex_op_read of the committed capture, 1M trials)."""
    sectors = _traffic(kernel, "l2_read_sectors_per_launch")
    if sectors is None:
        return None
    sectors *= trials / TRIALS_PER_GPU
    achieved = sectors / (kernel_ms / 1e3) / 1e9
    return {"sectors_per_launch": sectors, "achieved": achieved, "peak": SECTOR_PEAK_G_PER_S, "unit": "G sectors/s",
            "frac": achieved / SECTOR_PEAK_G_PER_S,
            "peak_source": "measured: scripts/micro/gather_rate.cu (random 16-byte L2 reads, nothing else running)",
            "note": "ids (125M sectors per 1M trials) and relay-record gathers share the SM's L2 read path; "
                    "this, not HBM bandwidth, bounds K2 (DESIGN.md section 4)"}


def roofline(trials: int, kernel_ms: float, kernel: str, packed_id_bytes: int | None = None) -> dict:
    """K2's roofline on the bytes that cross HBM (the verdict's rule: the
    lookups are served from L2 / shared memory by design, so the SURVEY 8(d)
    lookup-equivalent figure is reported separately, not as `frac`).
    `packed_id_bytes`: the launch streamed the packed resident ids
    (ARE_PACKED_IDS=1), so those bytes replace the uint32 ids."""
    peak, peak_src = _peaks()
    hbm = trials * compulsory_bytes_per_trial()
    formula = "trials x (4*E + 8 + 8): ids, offset, float64 YLT slot -- the bytes that cross HBM"
    if packed_id_bytes is not None:
        hbm = packed_id_bytes + trials * 16
        formula = ("packed ids (8 bytes per 3 ids, whole 96-id blocks) + trials x (8 + 8): offset, "
                   "float64 YLT slot -- the bytes that cross HBM")
        kernel = kernel + " (packed ids)"
    achieved = hbm / (kernel_ms / 1e3) / 1e9
    traffic = _traffic(kernel)
    lk = trials * bytes_per_trial()
    return {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
        "traffic": traffic, "traffic_ratio": (traffic / (hbm / (trials / TRIALS_PER_GPU))) if traffic else None,
        "kernel": kernel, "kernel_ms": kernel_ms, "bytes_per_launch": hbm,
        "bytes_formula": formula,
        "peak_source": peak_src,
        "traffic_note": "ncu dram__bytes_read+write per 1M-trial launch (profiles/k2_traffic.json); "
                        "traffic_ratio = traffic / bytes_per_launch at 1M trials",
        "sector_throughput": _sector_roofline(kernel, kernel_ms, trials),
        "lookup_equivalent": {
            "bytes_per_launch": lk, "formula": "trials x (12 + 4*E*(1+J)), SURVEY.md 8(d)",
            "gbs": lk / (kernel_ms / 1e3) / 1e9, "ratio_to_peak": lk / (kernel_ms / 1e3) / 1e9 / peak,
            "note": "one fp32 load per (event, ELT) lookup as if every lookup went to HBM; K2 skips the "
                    "86% of occurrences no ELT holds (bit-exact) and serves the rest from L2/shared "
                    "memory, so this exceeds 1 and is not a roofline fraction"},
    }


def _setup_dist():
    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device -- the B200 engine has no CPU fallback")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # ARE_BENCH_BACKEND=gloo lets several ranks share one GPU, to exercise the
    # multi-rank control flow on a one-GPU box (NCCL refuses duplicate GPUs)
    backend = os.environ.get("ARE_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group(backend, device_id=dev if backend == "nccl" else None)
    return world, rank, backend, local, dev


def _device_yet(first: int, last: int, dev, threads: int, chunk: int = 1 << 20):
    """The ids of trials [first, last) generated in host chunks straight into
    HBM (a 10M-trial shard is 40 GB; the host never holds more than a chunk)."""
    import torch

    from paper_1308_2066_b200.resident import DeviceYearEventTable

    n = last - first
    d_ids = torch.zeros(n * EVENTS + 4, dtype=torch.int32, device=dev)
    buf = np.empty(chunk * EVENTS, dtype=np.uint32)
    for a in range(first, last, chunk):
        b = min(last, a + chunk)
        y = bulk_chunk(a, b, threads, buf)
        d_ids[(a - first) * EVENTS:(b - first) * EVENTS].copy_(torch.from_numpy(y.view(np.int32)))
    offsets = np.arange(n + 1, dtype=np.int64) * EVENTS
    return DeviceYearEventTable.from_device(CATALOG, d_ids, torch.from_numpy(offsets).to(dev), offsets)


def bulk_chunk(a: int, b: int, threads: int, buf: np.ndarray) -> np.ndarray:
    from paper_1308_2066_b200.synth import bulk_yet

    return bulk_yet(SEED, CATALOG, a, b, EVENTS, threads=threads, out=buf).event_ids


def _pinned_host_yet(yet, local: int):
    import torch

    from paper_1308_2066_b200.portfolio import YearEventTable

    try:
        with GpuLocalCpus(local):
            ids = torch.from_numpy(yet.event_ids.view(np.int32)).pin_memory()
            offs = torch.from_numpy(np.ascontiguousarray(yet.offsets)).pin_memory()
        pinned = True
    except RuntimeError:  # page-locking refused (e.g. ulimit -l with 8 ranks): pageable, staged copies
        ids = torch.from_numpy(yet.event_ids.view(np.int32))
        offs = torch.from_numpy(np.ascontiguousarray(yet.offsets))
        pinned = False
    return YearEventTable(CATALOG, ids.numpy().view(np.uint32), None, offs.numpy()), pinned, (ids, offs)


def _stats(xs) -> dict:
    xs = [float(x) for x in xs]
    return {"median": float(np.median(xs)), "max": max(xs), "min": min(xs)} if xs else {}


def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_1308_2066_b200 import _native
    from paper_1308_2066_b200.direct_access import TableSet
    from paper_1308_2066_b200.distributed import allgather_portfolio, allgather_ylt, max_over_ranks, partition
    from paper_1308_2066_b200.engine import layer_pool, price_layer, simulate_layers_device
    from paper_1308_2066_b200.resident import DeviceYearEventTable
    from paper_1308_2066_b200.risk import order_stats, order_stats_async, rollup_device

    workload = args.workload
    world, rank, backend, local, dev = _setup_dist()
    threads = max(1, host_cores() // max(world, 1))
    strong = workload in ("c3", "c4")
    total_trials = {"c2": TRIALS_PER_GPU * world, "c3": TRIALS_PER_GPU, "c4": 10 * TRIALS_PER_GPU}[workload]
    t_gen = time.perf_counter()
    # global YET offsets are fixed-length, so the partition is computable without the ids
    g_offsets = np.arange(total_trials + 1, dtype=np.int64) * EVENTS
    parts = partition(g_offsets, world)
    t0, t1 = parts[rank]
    n_local = t1 - t0
    stream = torch.cuda.current_stream(dev)
    host_yet = None
    if workload == "c2":
        host_yet = make_yet(t0, t1, threads)
        dyet = DeviceYearEventTable(host_yet, device=local)
    else:
        dyet = _device_yet(t0, t1, dev, threads)
    gen_s = time.perf_counter() - t_gen

    if workload == "c3":
        layers = c3_portfolio()
        pool, masks = layer_pool(layers)
        tset = TableSet.from_elts(pool, CATALOG)
        lterms = [la.terms for la in layers]
        plan = tset.plan(*tset.selection_arrays(None), pool=True)
        info = _native.plan_info(plan)
        d_layers = torch.empty((16, n_local), dtype=torch.float64, device=dev)
        kernel_name = "k2_layers (16 layers fused)"
    else:
        layer = make_layer()
        tset = TableSet.from_elts(layer.elts, CATALOG)
        rows, rate, ret, lim, share = tset.selection_arrays(None)
        plan = tset.plan(rows, rate, ret, lim, share)
        info = _native.plan_info(plan)
        d_local = torch.empty(n_local, dtype=torch.float64, device=dev)
        kernel_name = "k2_hotset"

    def step(ev=None):
        """K2 over this rank's trials -> (N > 1) the YLT exchange -> K3."""
        if ev is not None:
            ev[0].record(stream)
        if workload == "c3":
            simulate_layers_device(dyet, tset, masks, lterms, out=d_layers, check=False)
        else:
            dyet.simulate_device(plan, layer.terms, out=d_local, stream=stream, check=False)
        if ev is not None:
            ev[1].record(stream)
        if workload == "c3":
            if world > 1:
                _, full = allgather_portfolio(list(d_layers), parts)
            else:
                full = rollup_device(list(d_layers))
        else:
            full = allgather_ylt(d_local, parts) if world > 1 else d_local
        if ev is not None:
            ev[2].record(stream)
        res = order_stats(full, RPS, stream=stream)
        if ev is not None:
            ev[3].record(stream)
        return res

    # Pipelined steps (c2, c4): step i's K2 runs on `stream` over all but k SMs
    # (ARE_SPARE_SMS(k)) while step i-1's exchange and K3 run on `side` over
    # the k spare SMs (2 CTAs each, no host wait), each step writing its own
    # YLT buffer (two, reused once the K3 that read them is done) and result
    # row.  k grows with the table K3 reads (this rank's YLT after the
    # exchange) relative to the trials K2 processes, so the overlapped K3
    # stays shorter than K2: 1 at N=1, N on N GPUs.  It pays while the YLT K3
    # streams stays small next to L2 (C2 on one GPU: 8 MB, +4%); with C4's
    # 80 MB YLT the overlapped K3 evicts K2's records from L2 and K2 slows by
    # more than K3 costs, so the headline steps stay sequential (--pipeline
    # times pipelined steps instead; the C2 line reports them beside).
    pipelined = workload != "c3" and args.pipeline
    can_pipeline = workload != "c3"
    spare = max(1, -(-(total_trials if world > 1 else n_local) // max(n_local, 1)))
    if can_pipeline:
        side = torch.cuda.Stream(dev)
        bufs = [d_local, torch.empty_like(d_local)]
        d_res = torch.zeros((args.warmup + args.steps, 16), dtype=torch.float64, device=dev)
        freed = [None, None]

        def pstep(i, ev):
            b = i & 1
            if freed[b] is not None:
                stream.wait_event(freed[b])  # the K3 that last read this buffer is done
            ev[0].record(stream)
            dyet.simulate_device(plan, layer.terms, out=bufs[b], stream=stream, check=False,
                                 flags=_native.spare_sms(spare))
            ev[1].record(stream)
            side.wait_event(ev[1])
            with torch.cuda.stream(side):
                full = allgather_ylt(bufs[b], parts) if world > 1 else bufs[b]
                ev[2].record(side)
                order_stats_async(full, RPS, d_res[i], side, max_ctas=2 * spare)
                ev[3].record(side)
            freed[b] = ev[3]

    if pipelined:
        wev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.warmup)]
        for i in range(args.warmup):
            pstep(i, wev[i])
    else:
        for _ in range(args.warmup):
            step()
    _native.check(_native.load().are_check_errors(plan.value, None))
    torch.cuda.synchronize(dev)
    if workload != "c3":
        info = _native.plan_info(plan)  # the relay records are built by the first launch
        kernel_name = "k2_relay" if info.relay else "k2_hotset"
    packed_bytes = None  # ARE_PACKED_IDS=1: the relay kernel streamed the packed resident ids
    if workload != "c3" and info.relay and getattr(dyet, "d_packed", None) is not None:
        packed_bytes = int(dyet.d_packed.numel()) * 8
    if world > 1:
        dist.barrier()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize(dev)
        start.record(stream)
        for i in range(args.steps):
            if pipelined:
                pstep(args.warmup + i, evs[i])
            else:
                pml_v, tvar_v = step(evs[i])
        if pipelined:
            stream.wait_event(evs[-1][3])  # the last step's K3
        stop.record(stream)
        torch.cuda.synchronize(dev)
    launches = _native.launch_count() - launches0
    pipelined_side = None
    if not pipelined and can_pipeline and world == 1 and workload == "c2":
        # the same steps pipelined, reported beside the sequential headline
        pev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.warmup + 20)]
        for i in range(args.warmup):
            pstep(i, pev[i])
        torch.cuda.synchronize(dev)
        p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        p0.record(stream)
        for i in range(args.warmup, args.warmup + 20):
            pstep(i % d_res.shape[0], pev[i])
        stream.wait_event(pev[-1][3])
        p1.record(stream)
        torch.cuda.synchronize(dev)
        pms = p0.elapsed_time(p1) / 20
        last = d_res[(args.warmup + 19) % d_res.shape[0]].cpu().numpy()
        assert list(last[: len(RPS)]) == list(pml_v), "pipelined and sequential K3 disagree"
        pipelined_side = {
            "value": total_trials / (pms / 1e3), "ms_per_step": pms, "spare_sms": spare,
            "k2_ms": float(np.mean([e[0].elapsed_time(e[1]) for e in pev[args.warmup:]])),
            "k3_overlapped_ms": float(np.mean([e[2].elapsed_time(e[3]) for e in pev[args.warmup:]])),
            "note": "the same steps pipelined (bench.py --pipeline): step i's K3 on the SM K2 leaves free "
                    "(are_order_stats_async, 2 CTAs, no host wait) overlaps step i+1's K2 on 147 SMs"}
    if pipelined:
        last = d_res[-1].cpu().numpy()
        pml_v, tvar_v = last[: len(RPS)], last[8: 8 + len(RPS)]
        # the same step run sequentially (K2 on every SM, then the blocking
        # order_stats), for the record
        seq_ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(10)]
        torch.cuda.synchronize(dev)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for i in range(10):
            seq_pml, _ = step(seq_ev[i])
        s1.record(stream)
        torch.cuda.synchronize(dev)
        assert list(seq_pml) == list(pml_v), "pipelined and sequential K3 disagree"
        sequential = {"ms_per_step": s0.elapsed_time(s1) / 10,
                      "k2_ms": float(np.mean([e[0].elapsed_time(e[1]) for e in seq_ev])),
                      "k3_ms": float(np.mean([e[2].elapsed_time(e[3]) for e in seq_ev])),
                      "note": "the same step without pipelining: K2 on all 148 SMs, then the exchange and "
                              "a blocking K3 on the full grid"}
    if world > 1:
        dist.barrier()
    elapsed_ms = start.elapsed_time(stop)
    k2_ms = float(np.mean([e[0].elapsed_time(e[1]) for e in evs]))
    xchg_ms = float(np.mean([e[1].elapsed_time(e[2]) for e in evs]))
    k3_ms = float(np.mean([e[2].elapsed_time(e[3]) for e in evs]))  # pipelined: on the spare SM, overlapped
    mx = (lambda v: max_over_ranks(v, dev)) if world > 1 else (lambda v: v)
    elapsed_max = mx(elapsed_ms)
    phases = {"k2_ms": mx(k2_ms), "exchange_ms": mx(xchg_ms), "k3_ms": mx(k3_ms),
              "exchange": ("allgather_portfolio (16 layer rows + portfolio, one NCCL all-gather)" if workload == "c3"
                           else "allgather_ylt (one NCCL all-gather)") if world > 1 else
              ("k3_rollup of the 16 layers" if workload == "c3" else "none (one GPU)")}
    if pipelined:
        phases["pipelined"] = (f"step i's exchange + K3 ({2 * spare} CTAs on the {spare} SM(s) K2 leaves free, stream "
                               f"`side`, no host wait) overlap step i+1's K2 (the other SMs); k3_ms is that overlapped "
                               f"K3's duration")
    value = total_trials * args.steps / (elapsed_max / 1e3)

    side = {}
    if workload == "c2":
        # ---- separately reported work unit: pre-combined plan
        pre_plan = tset.plan(rows, rate, ret, lim, share, precombine=True)
        for _ in range(3):
            dyet.simulate_device(pre_plan, layer.terms, out=d_local, stream=stream, check=False)
        pe = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        pe[0].record(stream)
        for _ in range(10):
            dyet.simulate_device(pre_plan, layer.terms, out=d_local, stream=stream, check=False)
        pe[1].record(stream)
        torch.cuda.synchronize(dev)
        pre_ms = pe[0].elapsed_time(pe[1]) / 10
        peak, _ = _peaks()
        side["precombined_k2"] = {
            "kernel_ms": pre_ms, "trials_per_s": n_local / (pre_ms / 1e3),
            "achieved_gbs": n_local * compulsory_bytes_per_trial() / (pre_ms / 1e3) / 1e9,
            "frac": n_local * compulsory_bytes_per_trial() / (pre_ms / 1e3) / 1e9 / peak,
            "note": "different unit of work (financial terms folded per event in K1); not the headline"}
        # ---- C3's fused 16-layer pass on this GPU
        side["c3_fused_layers"] = c3_fused(dyet, stream)
        # ---- the same K2 over the packed resident ids (opt-in layout)
        if packed_bytes is None and info.relay:
            side["packed_ids"] = packed_side(dyet, plan, layer.terms, d_local, stream, n_local,
                                             k2_ms, xchg_ms + k3_ms)

    # ---- e2e: the public host API on pinned host buffers --------------------
    # c2: this rank's whole shard; c3/c4: a bounded host sample of it (the
    # rate is linear in trials), said in the line
    e2e_trials = n_local if workload == "c2" else min(n_local, TRIALS_PER_GPU)
    src = host_yet if host_yet is not None else make_yet(t0, t0 + e2e_trials, threads)
    hyet, host_pinned, _keep = _pinned_host_yet(src, local)
    e_parts = partition(np.arange(e2e_trials * world + 1, dtype=np.int64) * EVENTS, world) if strong else parts
    ph = {"price_ms": [], "exchange_ms": [], "order_stats_ms": []}

    def e2e_step():
        from paper_1308_2066_b200.engine import run_aggregate_analysis
        from paper_1308_2066_b200.portfolio import YearEventTable

        a = time.perf_counter()
        if workload == "c3":
            # the entry point on a fresh host YET object every step (its promotion
            # cache must not skip the upload): H2D + K0 + fused K2-L + D2H
            y = YearEventTable(CATALOG, hyet.event_ids, None, hyet.offsets)
            ylts = run_aggregate_analysis(layers, y)
            local_rows = [torch.from_numpy(np.asarray(t.losses)).to(dev) for t in ylts]
        else:
            ylt, _ = price_layer(hyet, tset, None, layer.terms)
        b = time.perf_counter()
        if workload == "c3":
            full = allgather_portfolio(local_rows, e_parts)[1] if world > 1 else rollup_device(local_rows)
        elif world > 1:
            full = allgather_ylt(torch.from_numpy(ylt).to(dev), e_parts)
        else:
            full = ylt
        c = time.perf_counter()
        r = order_stats(full, RPS)
        d = time.perf_counter()
        ph["price_ms"].append((b - a) * 1e3)
        ph["exchange_ms"].append((c - b) * 1e3)
        ph["order_stats_ms"].append((d - c) * 1e3)
        return r

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    for _ in range(min(args.warmup, 2)):
        e2e_step()
    for k in ph:
        ph[k].clear()
    torch.cuda.synchronize(dev)
    rounds = []
    for _ in range(E2E_ROUNDS):
        if world > 1:
            dist.barrier()
        t_e2e = time.perf_counter()
        marks = [t_e2e]
        for _ in range(e2e_steps):
            e2e_step()
            marks.append(time.perf_counter())
        torch.cuda.synchronize(dev)
        secs = time.perf_counter() - t_e2e
        rounds.append((mx(secs), marks))
    e2e_s = float(np.median([r[0] for r in rounds]))
    per_step = [(b - a) * 1e3 for r in rounds for a, b in zip(r[1], r[1][1:])]
    e2e_value = e2e_trials * world * e2e_steps / e2e_s
    # the PCIe ceiling on this box: one plain pinned->device copy of the ids
    pinned_ids = _keep[0]
    d_probe = torch.empty(pinned_ids.numel(), dtype=torch.int32, device=dev)
    pcie = []
    for _ in range(3):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(stream)
        d_probe.copy_(pinned_ids, non_blocking=True)
        ev[1].record(stream)
        torch.cuda.synchronize(dev)
        pcie.append(pinned_ids.numel() * 4 / (ev[0].elapsed_time(ev[1]) / 1e3) / 1e9)
    del d_probe
    pcie_gbs = max(pcie)
    if workload == "c2" and world == 1:
        # the validated entry point on the same host YET:
        # run_aggregate_analysis promotes it to HBM (upload + K0 validation of
        # ids and trial lengths), then K1 + K2 + D2H; again on the same YET
        # object its validated device copy is reused
        from paper_1308_2066_b200.engine import run_aggregate_analysis_with_stats
        from paper_1308_2066_b200.portfolio import YearEventTable

        y = YearEventTable(CATALOG, hyet.event_ids, None, hyet.offsets)
        ep = []
        for _ in range(3):
            torch.cuda.synchronize(dev)
            t_ep = time.perf_counter()
            _, st_ep = run_aggregate_analysis_with_stats([layer], y)
            ep.append((time.perf_counter() - t_ep, st_ep.sim_seconds))
        side["entry_point"] = {
            "cold_s": ep[0][0], "repeat_s": min(e[0] for e in ep[1:]), "sim_s": min(e[1] for e in ep),
            "trials": e2e_trials,
            "note": "run_aggregate_analysis([layer], host YET of this rank): the first call uploads the 4 GB of "
                    "ids and validates them on the device (K0), later calls on the same YET object reuse "
                    "the validated device copy; the reference validates on the host (~9 s at C2)"}
        del y
    n_layers_out = 16 if workload == "c3" else 1
    h2d = int(hyet.event_ids.nbytes + hyet.offsets.nbytes + e2e_trials * 8 * n_layers_out)
    d2h = int(e2e_trials * 8 * n_layers_out + 2 * 8 * len(RPS))

    if rank != 0:
        dist.destroy_process_group()
        return

    name = {"c2": WORKLOAD, "c3": WORKLOAD_C3, "c4": WORKLOAD_C4}[workload]
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "trials/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": elapsed_max / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "vs_paper_c2075": value / 50_000.0 if workload == "c2" else None,
        "dtype": "f64",
        "data": "synthetic",
        "config": {
            "workload": name, "trials_total": total_trials, "trials_per_gpu": n_local,
            "events_per_trial": EVENTS, "catalog": CATALOG,
            "elts": 32 if workload == "c3" else N_ELTS, "layers": 16 if workload == "c3" else 1,
            "layer_terms": "C3 generator terms (PO XL / Agg XL alternating)" if workload == "c3" else list(TERMS),
            "return_periods": RPS,
            "parallelism": f"trial-sharded x{world} (split_by_events)" + (
                f", YLT all-gather over {backend.upper()}" if world > 1 else ""),
            "l2": "no flush: 4 GB id stream per 1M trials > 126 MB L2; hot-set records L2-resident by design",
            "generator": "ELTs: reference generator restatement seed 2066; YET: synth.bulk_yet",
            "kernel": kernel_name,
        },
        "phases_max_over_ranks": phases,
        **({"sequential": sequential} if pipelined else {}),
        **({"pipelined": pipelined_side} if pipelined_side else {}),
        "roofline": roofline(n_local, phases["k2_ms"], kernel_name, packed_bytes) if workload != "c3" else dict(
            roofline(n_local, phases["k2_ms"], kernel_name),
            bytes_per_launch=n_local * (compulsory_bytes_per_trial() + 8 * 15),
            achieved=n_local * (compulsory_bytes_per_trial() + 8 * 15) / (phases["k2_ms"] / 1e3) / 1e9,
            frac=n_local * (compulsory_bytes_per_trial() + 8 * 15) / (phases["k2_ms"] / 1e3) / 1e9 / _peaks()[0],
            bytes_formula="trials x (4*E + 8 + 16*8): ids and offset once, 16 float64 YLT rows"),
        "e2e": {"value": e2e_value, "unit": "trials/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_s * 1e3 / e2e_steps, "steps": e2e_steps, "trials_per_gpu": e2e_trials,
                "rounds_ms_per_step": [round(r[0] * 1e3 / e2e_steps, 2) for r in rounds],
                "step_ms": [round(x, 2) for x in per_step],
                "median_step_ms": float(np.median(per_step)),
                "phases_ms": {k: _stats(v) for k, v in ph.items()},
                "note": f"value = trials over the median of {E2E_ROUNDS} rounds of `steps` steps (every step timed, "
                        "H2D/D2H included); phases_ms split each step into the host API call that streams the "
                        "ids and runs K2 (price_layer / run_aggregate_analysis), the YLT exchange, and "
                        "order_stats (H2D of the YLT + K3)" + ("" if workload == "c2" else
                        f"; a {e2e_trials}-trial host sample per GPU (rate linear in trials)"),
                "h2d_gbs": h2d / (e2e_s / e2e_steps) / 1e9,
                "pcie_h2d_gbs_measured": pcie_gbs,
                "frac_of_pcie": h2d / (e2e_s / e2e_steps) / 1e9 / pcie_gbs,
                "host_pinned": host_pinned,
                "path": ("run_aggregate_analysis(16 layers, host YET)" if workload == "c3" else
                         "price_layer(pinned host YET) -> are_simulate_host") + " -> order_stats"},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(),
        "hot_set": {"hot_events": info.hot_events, "entries": info.entries,
                    "overflow_entries": info.overflow_entries, "filter_bits": info.filter_bits,
                    "smem_bytes": info.smem_bytes, "relay": bool(info.relay),
                    "relay_filter_bits": info.relay_filter_bits, "relay_smem_bytes": info.relay_smem_bytes},
        **side,
        "pml": list(map(float, pml_v)), "tvar": list(map(float, tvar_v)),
        "setup_seconds": {"generate": gen_s},
    }
    if world == 1 and workload == "c2" and not args.no_cpu_baseline:
        # min of 3 rounds, at W = all host cores and W = 1
        cores = host_cores()
        sample = args.cpu_sample or calibrate_sample(layer, cores, 4.0)
        cb = cpu_reference(layer, host_yet, sample, cores, steps=3)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        sample1 = args.cpu_sample or calibrate_sample(layer, 1, 3.0)
        cb1 = cpu_reference(layer, host_yet, sample1, 1, steps=3)
        line["cpu_baseline"]["w1"] = {k: cb1[k] for k in ("value", "unit", "cores", "sample")}
        line["cpu_baseline"]["host"] = host_descriptor()
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--cpu-sample", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-full-pass", action="store_true", help="reference arm: skip the one full 1M-trial pass")
    ap.add_argument("--pipeline", action="store_true",
                    help="time pipelined steps: step i's exchange + K3 on the SMs K2 leaves free overlap "
                         "step i+1's K2 (default: one step after another)")
    ap.add_argument("--workload", choices=["c2", "c3", "c4"], default="c2",
                    help="c2: 1M trials per GPU (weak scaling, the headline); c3: the 16-layer portfolio over "
                         "1M trials split across the GPUs; c4: 10M trials split across the GPUs")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="strong = --workload c4 (C4's fixed 10M trials over N GPUs)")
    ap.add_argument("--packed-ids", action="store_true",
                    help="keep the resident ids in the packed layout (ARE_PACKED_IDS=1): the relay kernel "
                         "streams 2/3 of the id bytes; roofline bytes follow (default: uint32 ids, the packed "
                         "K2 is reported beside as `packed_ids`)")
    args = ap.parse_args()
    if args.packed_ids:
        os.environ["ARE_PACKED_IDS"] = "1"
    if args.scaling == "strong" and args.workload == "c2":
        args.workload = "c4"
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
