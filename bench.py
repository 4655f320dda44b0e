#!/usr/bin/env python
"""ICQ query-path benchmark on B200 — prints ONE JSON line (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

Workload: one BASELINE config (default c5 = configs[4], the largest
single-GPU config: 100M items, batch 512; c1..c5 selectable with --config),
seeded synthetic data (tools/workloads.py), books trained by the reference
(bench_data/), database encoded on the GPU.  A step = one batch of queries
through the hot path (K1 LUT build + fused scan/prune/refine/top-k kernel).

value    queries/s over all ranks, device time (CUDA events on the launch
         stream), inputs resident in HBM, L2 flushed before every step
e2e      queries/s through the C-ABI host-buffer call (icq_search_host):
         pinned host queries -> H2D -> search -> D2H of ids/scores/refinements
roofline effective code-stream bandwidth of the scan kernel:
         (batch * n * |F| fast-code bytes) / scan-kernel time, vs the measured
         HBM copy peak (MEASURED_PEAKS.json)
cpu_baseline the reference algorithm's CPU port (oracle.two_step_loop, a
         literal restatement of search.py:112-165) on a bounded query sample,
         as many host processes as cores and RAM allow, rank 0 at N=1.
sigma_sweep  the same batch pipeline at sigma in {mean lambda, 4 mean lambda,
         learned}: q/s, refined fraction, list (filter pass) fraction, items
         walked in order, recall@k against the exact engine.
Multi-GPU: query batches are independent -> replicas, no collective
(scaling "weak": each rank runs the same number of batches).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from tools.workloads import CONFIGS, SEED_DB, SEED_QUERIES, SEED_TRAIN  # noqa: E402


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        z = json.loads(p.read_text())
        return float(z["hbm_gbs"]), float(z.get("sm_max_mhz", 1965.0)), "measured"
    return 6650.0, 1965.0, "fallback"


def _profiled_traffic(cfg: str):
    """DRAM bytes per scan-kernel launch (dram__bytes_read.sum + write.sum) from
    the committed ncu --set full summary of this config, scaled to the bench
    batch; None when no capture is committed."""
    p = ROOT / "profiles" / "traffic.json"
    if not p.exists():
        return None
    z = json.loads(p.read_text()).get(cfg)
    return None if z is None else z.get("dram_bytes_per_launch_at_bench_batch")


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons during the timed region,
    sampled in-process through NVML every 250 ms, plus one sample taken while
    the last steps still run.  (An `nvidia-smi -lms 20` child, the first
    version, stalled the launch path for 5-70 ms in about half of the c4
    runs; in-process NVML queries every 20 ms still cost the long c5 kernels
    ~6-18 % -- 91-103 ms per step against 86 ms without the sampler -- so the
    sampler now runs at 4 Hz.)"""

    NAMES = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
             ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.rows = []  # (sm MHz, max sm MHz, reason bits)
        self._stop = threading.Event()
        self._t = None
        self.recording = False  # rows are kept only while the timed region runs
        self.periodic = True    # sample from the thread during the timed region
        self._first = threading.Event()
        self._nv = None
        self._h = None

    def _handle(self):
        import pynvml as nv
        nv.nvmlInit()
        self._nv = nv
        try:  # the NVML device of this CUDA device (CUDA_VISIBLE_DEVICES may remap)
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        if os.environ.get("ICQ_BENCH_NO_CLOCKS"):  # (diagnostics: timing without the sampler)
            return self
        try:
            self._h = self._handle()
            self._mx = self._nv.nvmlDeviceGetMaxClockInfo(self._h, self._nv.NVML_CLOCK_SM)
        except Exception:
            self._h = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rb = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                break
            self._first.set()
            if self.recording:
                self.rows.append((float(sm), float(self._mx), int(rb)))
            self._stop.wait(0.25)
            # launch-bound steps (a few ms, two dozen launches each): an NVML
            # query now and then holds a driver lock for 25-110 ms and shows up
            # as one slow step -- such runs are sampled from the main thread
            # only (sample_now: before the timed region and while its last
            # steps still run)
            while self.recording and not self.periodic and not self._stop.is_set():
                self._stop.wait(0.05)

    def sample_now(self):
        """One sample from the calling thread (short timed regions: taken
        while the enqueued steps still run)."""
        if self._h is None:
            return
        try:
            sm = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
            rb = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            self.rows.append((float(sm), float(self._mx), int(rb)))
        except Exception:
            pass

    def wait_started(self, timeout=10.0):
        if self._t is not None:
            self._first.wait(timeout)

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({nm for r in self.rows for nm, bit in self.NAMES if r[2] & bit})
        return {"sm_mhz": float(np.median([r[0] for r in self.rows])),
                "sm_max_mhz": max(r[1] for r in self.rows), "reasons": reasons,
                "samples": len(self.rows), "source": "NVML, 250 ms"}


# ---------------------------------------------------------------------------
# CPU baseline: the reference algorithm on host cores
# ---------------------------------------------------------------------------
_CPU = {}


def _cpu_one(qi):
    from oracle import icq_oracle as O

    c = _CPU
    t0 = time.perf_counter()
    r = O.two_step_loop(c["books"], c["codes"], c["fast"], c["sigma"], c["Q"][qi], c["k"])
    return qi, r.ids, r.scores, r.ops.refinements, time.perf_counter() - t0


def cpu_workers(w, cap=None):
    """Host processes for the CPU port: every core, bounded by RAM -- each
    in-flight query materialises (n, K) gathers plus two Python lists of n
    floats (search.py:94, :146-147), ~ n * (16 K + 80) bytes."""
    import psutil

    cores = os.cpu_count() or 1
    per_q = w.n * (16 * w.K + 80)
    avail = psutil.virtual_memory().available - (8 << 30)
    by_ram = max(1, int(avail // per_q))
    n = min(cores, by_ram)
    return min(n, cap) if cap else n


def cpu_baseline(books, codes_host, fast, sigma, Qhost, k, nq, workers):
    import multiprocessing as mp

    _CPU.update(books=books, codes=codes_host, fast=fast, sigma=sigma, Q=Qhost, k=k)
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(workers) as pool:
        res = pool.map(_cpu_one, range(nq), chunksize=1)
    wall = time.perf_counter() - t0
    return res, wall


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=os.environ.get("ICQ_BENCH_CONFIG", "c5"),
                    choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--sigma", type=float, default=None, help="override the learned margin")
    ap.add_argument("--sweeps", type=int, default=10, help="ICM sweeps when encoding the database")
    ap.add_argument("--cpu-queries", type=int, default=0, help="CPU baseline sample (0 = auto)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the sigma sweep")
    ap.add_argument("--sweep-steps", type=int, default=3)
    args = ap.parse_args()

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference" and rank != 0:
        return 0  # the CPU reference arm runs on rank 0 only
    torch.cuda.set_device(local)
    dist = None
    if world > 1 and args.impl == "b200":
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from tools.workloads import build_database, index_rule, load_books, queries

    w = CONFIGS[args.config]
    books, meta = load_books(w)
    fast, sigma, rule, sigma_rule = index_rule(w, meta, args.sigma)

    t0 = time.time()
    enc_stats = {}
    codes = build_database(w, books, sweeps=args.sweeps, stats=enc_stats)
    Qall = queries(w)
    torch.cuda.synchronize()
    prep_s = time.time() - t0
    B = w.batch
    nbatches = (w.Q + B - 1) // B

    base_config = {
        "workload": f"{w.name}: n={w.n} d={w.d} K={w.K} m=256 |F|={w.F} k={w.k} "
                    f"queries={w.Q} batch={B} dist={w.dist}",
        "n": w.n, "d": w.d, "K": w.K, "m": 256, "F": w.F, "k": w.k, "batch": B,
        "fast": fast.tolist(), "fast_rule": rule, "sigma": sigma, "sigma_rule": sigma_rule,
        "books": f"reference icq.train on {int(meta['train_rows'])} seeded rows, "
                 f"{int(meta['epochs'])} epoch(s), seed {int(meta['seed'])}",
        "seeds": {"train": SEED_TRAIN, "db": SEED_DB, "queries": SEED_QUERIES},
        "encode": (f"GPU float64 ICM encoder (icq_encode: reference assign_codes, greedy + "
                   f"<= {args.sweeps} sweeps; {enc_stats.get('sweeps_used')} used; "
                   f"{enc_stats.get('encode_seconds', 0):.1f} s for {w.n} rows)"),
        "l2": "flushed (256 MiB write) before every timed step",
        "parallelism": f"replicas{world}" if world > 1 else "single",
    }

    if args.impl == "reference":
        return run_reference(args, w, books, codes, fast, sigma, Qall, base_config)

    import paper_1912_08756_b200 as icqb

    dev = icqb.DeviceIndex.from_device(books, codes, fast)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    from paper_1912_08756_b200.replicas import aggregate, rank_batch

    def batch(i):
        b = rank_batch(rank, world, i, nbatches)
        return Qall[b * B:(b + 1) * B]

    def step(i, ev=None):
        qb = batch(i)
        flush.zero_()
        if ev:
            ev[0].record(stream)
        lut = dev.build_lut_device(qb)
        if ev:
            ev[1].record(stream)
        out = dev.search_lut_device(lut, w.k, sigma, stats=True)
        if ev:
            ev[2].record(stream)
        return qb.shape[0], out

    clk = ClockSampler(local).__enter__()
    clk.wait_started()
    for i in range(args.warmup):
        if i == args.warmup - 1:  # (the first steps pay one-time allocations)
            torch.cuda.synchronize()
            # one clock sample under load right before the timed region (an NVML
            # query can delay the launches that follow it by tens of ms: it is
            # taken here, ahead of the last warm-up step, not inside the region)
            clk.sample_now()
            t_w = time.perf_counter()
        step(i)
    torch.cuda.synchronize()
    clk.periodic = args.warmup > 0 and (time.perf_counter() - t_w) > 0.02
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    outs = []
    L = icqb._native.lib()
    L.icq_profile_read(None, None)  # drop anything recorded during warm-up
    L.icq_profile_enable(1)  # CUDA events around each pipeline kernel, launch stream
    launches0 = int(L.icq_kernel_launches())
    clk.recording = True
    for i in range(args.steps):
        outs.append(step(args.warmup + i, evs[i]))
    clk.sample_now()  # the last steps are still running on the device
    torch.cuda.synchronize()
    gpu_launches = int(L.icq_kernel_launches()) - launches0  # this library's kernels, timed region
    clk.recording = False
    clk.__exit__(None, None, None)
    L.icq_profile_enable(0)
    import ctypes as _C

    kms = (_C.c_double * 5)()
    klaunch = _C.c_int32()
    L.icq_profile_read(kms, _C.byref(klaunch))
    t_pro_k, t_filter_k, t_replay_k, t_count_k, t_refine_k = (x / 1e3 for x in kms)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = sorted(e[0].elapsed_time(e[2]) for e in evs)
    t_lut = sum(e[0].elapsed_time(e[1]) for e in evs) / 1e3
    t_scan = sum(e[1].elapsed_time(e[2]) for e in evs) / 1e3
    t_total = t_lut + t_scan
    nq = sum(o[0] for o in outs)
    refine = torch.cat([o[1]["refinements"] for o in outs]).double()
    stats = torch.cat([o[1]["stats"] for o in outs]).double()
    nq_all, (t_total, t_scan, t_lut) = aggregate(dist, "cuda", nq, [t_total, t_scan, t_lut])
    qps = nq_all / t_total
    lookups = nq * w.n * w.F
    # the filter kernel streams the fast codes of items [P, n) of every query
    p_mean = float(stats[:, 3].mean().item())
    # items the filter streamed: after the prologue, minus the tails of slices
    # that overflowed their candidate pages (the replay rescans those instead)
    skipped = float(stats[:, 15].sum().item())
    filter_bytes = (nq * (w.n - p_mean) - skipped) * w.F
    filter_gbs = filter_bytes / t_filter_k / 1e9  # per-GPU filter kernel (this rank)
    hbm_peak, sm_max, peak_kind = _peaks()
    # shared-memory gather peak: conflict-free lane-private LDS.32 measured at
    # 0.715 warp instructions / clock / SM on this pool's B200s (tools/lds_peak.cu,
    # profiles/r02_lds_peak.txt); the nominal crossbar rate is 1.0
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    smem_nominal_glps = sms * 32 * sm_max * 1e6 / 1e9
    smem_peak_glps = 0.715 * smem_nominal_glps

    # e2e through the C-ABI host-buffer call (pinned host queries)
    e2e = None
    if not args.no_e2e:
        Qpin = torch.empty((B, w.d), dtype=torch.float64, pin_memory=True)
        e2e_t = 0.0
        e2e_n = 0
        for i in range(args.warmup + args.steps):
            qb = batch(i)
            Qpin[:qb.shape[0]].copy_(qb.cpu())
            qh = Qpin[:qb.shape[0]].numpy()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.search_host(qh, w.k, sigma, exact=False)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                e2e_t += dt
                e2e_n += qb.shape[0]
        e2e_all, (e2e_tmax,) = aggregate(dist, "cuda", e2e_n, [e2e_t])
        e2e_rate = e2e_all / e2e_tmax
        e2e = {"value": e2e_rate, "unit": "queries/s", "h2d_bytes_per_step": B * w.d * 8,
               "d2h_bytes_per_step": B * w.k * 16 + B * 8,
               "path": "icq_search_host (C ABI, host buffers)"}

    # recall of two-step vs exact engine + parity sample vs the CPU reference port
    qb = batch(0)
    two = dev.search_device(qb, w.k, sigma)
    ex = dev.search_device(qb, w.k, exact=True)
    torch.cuda.synchronize()
    ti, ei = two["ids"].cpu().numpy(), ex["ids"].cpu().numpy()
    recall = float(np.mean([np.isin(ti[i], ei[i]).mean() for i in range(ti.shape[0])]))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        codes_h = codes.cpu().numpy()
        workers = cpu_workers(w)
        # one query per process, at least 8 queries (two rounds on small hosts)
        nqc = args.cpu_queries or (max(8, workers) if w.n < 50_000_000 else workers)
        Qh = Qall[:nqc].cpu().numpy()
        res, wall = cpu_baseline(books, codes_h, fast, sigma, Qh, w.k, nqc, min(workers, nqc))
        ids, sc, rf, _ = dev.search_host(Qh, w.k, sigma, exact=False)
        mism = sum(int(not (np.array_equal(ids[qi], r_ids) and np.array_equal(sc[qi], r_sc)
                            and rf[qi] == r_rf)) for qi, r_ids, r_sc, r_rf, _ in res)
        cpu = {"value": nqc / wall, "unit": "queries/s", "cores": min(workers, nqc), "kind": "port",
               "sample": f"{nqc} queries of {w.name} (first {nqc} of the query set), oracle."
                         f"two_step_loop (literal search.py:112-165), {min(workers, nqc)} processes",
               "cpu_seconds": sum(r[4] for r in res),
               "parity_vs_gpu": {"queries": nqc, "mismatches": mism}}
        del codes_h

    sweep = None
    if not args.no_sweep:
        sweep = sigma_sweep(args, w, dev, meta, sigma, batch, flush, stream, ex, Qall)

    line = {
        "metric": "queries/sec (top-k two-step ICQ search); G code-lookups/s; fast-scan GB/s vs roofline",
        "value": qps,
        "unit": "queries/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": t_total / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u8 codes / f32 scan / f64 certified scores",
        "data": "synthetic (seeded; BASELINE names no dataset)",
        "config": base_config,
        "glookups_per_s": nq_all * w.n * w.F / t_total / 1e9,
        "lut_ms_per_step": t_lut / args.steps * 1e3,
        "step_ms_median_max": [step_ms[len(step_ms) // 2], step_ms[-1]],
        "scan_ms_per_step": t_scan / args.steps * 1e3,
        "pruning": {"refined_fraction": float(refine.mean().item() / w.n),
                    "insertions_per_query": float(stats[:, 0].mean().item()),
                    "prologue_insertions_per_query": float(stats[:, 10].mean().item()),
                    "replay_live_candidates_per_query": float(stats[:, 1].mean().item()),
                    "walked_items_per_query": float(stats[:, 2].mean().item()),
                    "walked_items_max_query": float(stats[:, 2].max().item()),
                    "rounds_per_query": float((stats[:, 7].long() >> 8).double().mean().item()),
                    "prologue_items_per_query": float(stats[:, 3].mean().item()),
                    "prologue_cycles_per_query": float(stats[:, 4].mean().item()),
                    "replay_cycles_per_query": float(stats[:, 5].mean().item()),
                    "replay_cycles_max_query": [float(stats[:, 5].max().item()), int(stats[:, 5].argmax().item()),
                                                float(stats[stats[:, 5].argmax(), 9].item()),
                                                float(stats[stats[:, 5].argmax(), 3].item())],
                    "rescanned_slices": int((stats[:, 6].long() & 0xFFFFF).sum().item()),
                    "overflow_slices_pages": int(((stats[:, 6].long() >> 20) & 0xFFFFF).sum().item()),
                    "overflow_slices_pool": int((stats[:, 6].long() >> 40).sum().item()),
                    "wide_queries": int((stats[:, 7].long() & 0xFF).sum().item()),
                    "prologue_f64_scored_per_query": float(stats[:, 8].mean().item()),
                    "filter_candidates_per_query": float(stats[:, 9].mean().item()),
                    "refine_inputs_per_query": float(stats[:, 11].mean().item()),
                    "refine_inputs_max_query": float(stats[:, 11].max().item()),
                    "filter_skipped_items_per_query": float(stats[:, 15].mean().item()),
                    "filter_pass_fraction": float(stats[:, 9].mean().item() / w.n),
                    "prologue_phase_cycles_per_query": {
                        "prefilter": float(stats[:, 12].mean().item()),
                        "score": float(stats[:, 13].mean().item()),
                        "decide": float(stats[:, 14].mean().item())},
                    "recall_vs_exact": recall},
        "roofline": {"bound": "hbm", "achieved": filter_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": filter_gbs / hbm_peak, "traffic": _profiled_traffic(w.name),
                     "peak_kind": peak_kind,
                     "kernel": "icq_filter_kernel (K3: fast-code stream, fp32 gather, compaction)",
                     "algorithmic_bytes_per_launch": filter_bytes / args.steps,
                     "filter_ms_per_launch": t_filter_k / args.steps * 1e3,
                     "filter_share_of_step": t_filter_k / t_total,
                     # the kernel's own bound: F table gathers per streamed item
                     "gather": {"glookups_per_s": filter_bytes / t_filter_k / 1e9,
                                "peak_measured": smem_peak_glps, "peak_nominal": smem_nominal_glps,
                                "frac_of_measured": (filter_bytes / t_filter_k / 1e9) / smem_peak_glps,
                                "count_kernel_frac_of_measured":
                                    (None if t_count_k <= 0 else
                                     (nq * (w.n - p_mean) * w.F / t_count_k / 1e9) / smem_peak_glps)}},
        "kernels_ms_per_step": {"lut": t_lut / args.steps * 1e3,
                                "prologue": t_pro_k / args.steps * 1e3,
                                "filter": t_filter_k / args.steps * 1e3,
                                "refine": t_refine_k / args.steps * 1e3,
                                "replay": t_replay_k / args.steps * 1e3,
                                "count": t_count_k / args.steps * 1e3},
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "cpu_baseline": cpu,
        "sigma_sweep": sweep,
        "setup_seconds": prep_s,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def sigma_sweep(args, w, dev, meta, sigma0, batch, flush, stream, ex, Qall):
    """The batch pipeline at the other operating points of SURVEY §8(d) rule
    step 4: sigma in {mean lambda, 4 mean lambda} and the learned margin
    (when it differs).  Device-timed like the headline (L2 flushed), one
    JSON object per sigma; recall@k against the exact engine on batch 0."""
    import torch

    lam = float(np.asarray(meta["lambdas"], dtype=np.float64).mean())
    learned = float(meta["learned_sigma"])
    pts = [("mean_lambda", lam), ("4_mean_lambda", 4 * lam)]
    if learned not in (0.0, sigma0, lam, 4 * lam):
        pts.append(("learned", learned))
    if sigma0 != 0.0:
        pts.insert(0, ("zero", 0.0))
    ei = ex["ids"].cpu().numpy()
    out = []
    for label, sg in pts:
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.sweep_steps)]
        res = []
        for i in range(1 + args.sweep_steps):  # one warm-up
            qb = batch(i)
            flush.zero_()
            if i:
                evs[i - 1][0].record(stream)
            lut = dev.build_lut_device(qb)
            o = dev.search_lut_device(lut, w.k, sg, stats=True)
            if i:
                evs[i - 1][1].record(stream)
                res.append((qb.shape[0], o))
        torch.cuda.synchronize()
        t = sum(a.elapsed_time(b) for a, b in evs) / 1e3
        nq = sum(r[0] for r in res)
        st = torch.cat([r[1]["stats"] for r in res]).double()
        rf = torch.cat([r[1]["refinements"] for r in res]).double()
        two = dev.search_device(batch(0), w.k, sg)
        ti = two["ids"].cpu().numpy()
        recall = float(np.mean([np.isin(ti[i], ei[i]).mean() for i in range(ti.shape[0])]))
        out.append({"sigma": sg, "label": label, "queries_per_s": nq / t,
                    "ms_per_step": t / args.sweep_steps * 1e3,
                    "refined_fraction": float(rf.mean().item() / w.n),
                    "list_fraction": float(st[:, 9].mean().item() / w.n),
                    "walked_items_per_query": float(st[:, 2].mean().item()),
                    "recall_at_k_vs_exact": recall, "steps": args.sweep_steps})
    return out


def run_reference(args, w, books, codes, fast, sigma, Qall, base_config):
    """--impl reference: the reference algorithm's CPU port on host cores
    (one query per process; as many processes as cores and RAM allow)."""
    codes_h = codes.cpu().numpy()
    # (n >= 50M: <= 8 processes, ~15 s per step, so 25 steps fit the driver's limit)
    workers = cpu_workers(w, cap=8 if w.n >= 50_000_000 else None)
    nq = args.cpu_queries or workers
    workers = min(workers, nq)
    Qh = Qall.cpu().numpy()
    rates = []
    for i in range(args.warmup + args.steps):
        sel = Qh[(i * nq) % w.Q:(i * nq) % w.Q + nq]
        res, wall = cpu_baseline(books, codes_h, fast, sigma, sel, w.k, sel.shape[0], workers)
        if i >= args.warmup:
            rates.append((sel.shape[0], wall))
    tot_q = sum(r[0] for r in rates)
    tot_t = sum(r[1] for r in rates)
    v = tot_q / tot_t
    line = {
        "impl": "reference",
        "metric": "queries/sec (top-k two-step ICQ search); G code-lookups/s; fast-scan GB/s vs roofline",
        "value": v, "unit": "queries/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded)", "config": base_config,
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": workers, "kind": "port",
                         "sample": f"{nq} queries per step, oracle.two_step_loop "
                                   f"(literal search.py:112-165), {workers} processes"},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
