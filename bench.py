#!/usr/bin/env python
"""Benchmark of the B200 two-pass DTW k-NN engine.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]

One STEP = one full pass of the hot path (query envelopes, LB_Keogh over the
whole database, LB_Improved on survivors, banded DTW, top-k, and for N > 1 the
NCCL all-gather + shard merge) over the whole workload of the config, with the
inputs resident in HBM.  Metric: query-candidate pairs/s (BASELINE.json); DTW
cells/s is reported beside it.  For N > 1 (torchrun) each rank owns a
contiguous shard of the database (total work fixed: strong scaling); time is
the max over ranks of CUDA-event time on the launching stream.

`--impl reference` times the fp64 CPU oracle (the paper's Algorithm 3 scan,
oracle/) on this box's host cores over a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        if os.environ.get("DTWLB_BENCH_NO_CLOCKS") == "1":  # (interference experiments only)
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", os.environ.get("DTWLB_BENCH_CLOCK_MS", "200")], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": mx, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- CPU oracle
def oracle_sample(cfg, qs, db, budget_s=15.0, threads=None):
    """Time the fp64 oracle (Alg. 3 scan, as it stands) on a bounded query sample."""
    import oracle
    threads = threads or os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.nn_twopass(qs[:1], db, cfg.w, cfg.p, cfg.k, threads=1)
    per_q = max(time.perf_counter() - t0, 1e-3)
    nq = int(max(1, min(len(qs) - 1, round(budget_s * threads / per_q))))
    nq = max(threads, nq // threads * threads) if nq >= threads else nq
    nq = min(nq, len(qs) - 1)
    t0 = time.perf_counter()
    oracle.nn_twopass(qs[1:1 + nq], db, cfg.w, cfg.p, cfg.k, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": nq * len(db) / dt, "unit": "pairs/s", "cores": min(threads, nq), "kind": "oracle",
            "sample": f"{nq} of {cfg.Q} queries x all {len(db)} database series (Alg. 3 fp64 scan, "
                      f"{min(threads, nq)} threads, {dt:.1f} s)", "seconds": dt,
            "single_thread": {"value": len(db) / per_q, "unit": "pairs/s",
                              "sample": f"query 0 x all {len(db)} series, 1 thread, {per_q:.2f} s"},
            "cpu_model": _cpu_model(), "host_threads": os.cpu_count()}


def _cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, cfg):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    qs, db = datagen.make(cfg)
    threads = os.cpu_count() or 1
    import oracle
    t0 = time.perf_counter()
    oracle.nn_twopass(qs[:1], db, cfg.w, cfg.p, cfg.k, threads=1)
    per_q = max(time.perf_counter() - t0, 1e-3)
    # bounded sample per step: ~20 s of wall time over all cores for K+W steps
    per_step_s = max(2.0, 150.0 / max(1, args.steps + args.warmup))
    nq = int(max(1, min(cfg.Q, round(per_step_s * threads / per_q))))
    times = []
    for s in range(args.warmup + args.steps):
        lo = (s * nq) % max(1, cfg.Q - nq)
        t0 = time.perf_counter()
        oracle.nn_twopass(qs[lo:lo + nq], db, cfg.w, cfg.p, cfg.k, threads=threads)
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    dt = statistics.mean(times)
    value = nq * cfg.N / dt
    line = {"impl": "reference", "metric": "query-candidate pairs/s (exact DTW k-NN)", "value": value,
            "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "Q": cfg.Q, "N": cfg.N, "n": cfg.n, "w": cfg.w, "p": cfg.p,
                       "k": cfg.k, "sample_queries_per_step": nq},
            "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": min(threads, nq), "kind": "oracle",
                             "sample": f"{nq} of {cfg.Q} queries x {cfg.N} series per step"},
            "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def run_ours(args, cfg):
    import torch
    import torch.distributed as dist
    from paper_0811_3301_b200 import binding as B
    from paper_0811_3301_b200.sharded import shard_range

    ws, rank, local = _dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if ws > 1 else 0)
    torch.cuda.set_device(dev)
    st = torch.cuda.current_stream()
    qshard = args.shard == "queries" and ws > 1  # comparison mode: replicated database, queries split
    lo, hi = shard_range(cfg.N, ws, rank) if not qshard else (0, cfg.N)
    qs_h, _ = datagen.make(cfg, N=0)
    db_h = datagen.series(cfg.family, hi - lo, cfg.n, cfg.seed, datagen.ROLE_DB, cfg.znorm, start=lo)
    qs = torch.from_numpy(qs_h).to(dev)
    db = torch.from_numpy(db_h).to(dev)
    k = cfg.k
    from paper_0811_3301_b200.sharded import make_communicator, sharded_nn_search
    # database-sharded N > 1: the library's own NCCL communicator does the threshold exchange
    # inside nn_search (no Python callback in the search loop); --py-exchange keeps the callback
    comm = make_communicator(device=dev) if ws > 1 and not qshard and not args.py_exchange else None
    idx = torch.empty((cfg.Q, k), dtype=torch.int64, device=dev)
    dst = torch.empty((cfg.Q, k), dtype=torch.float32, device=dev)
    gbufs = (torch.empty((ws * cfg.Q, k), dtype=torch.int64, device=dev),
             torch.empty((ws * cfg.Q, k), dtype=torch.float32, device=dev))
    last = {}
    # few queries (Q <= 8, n % 4 == 0): nn_search's streaming bound pass (no pre-filter)
    stream_mode = cfg.Q <= 8 and cfg.n % 4 == 0 and not args.no_stream
    pf = not args.no_prefilter and not stream_mode  # the piecewise-sum pre-filter runs
    db_env, index_ms = None, None
    if args.db_index:  # the database index (envelopes of the rows), built once outside the timed region
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        U_, L_ = B.lb_envelope(db, cfg.w)
        db_env = torch.stack([U_, L_]).contiguous()
        e1.record(st)
        torch.cuda.synchronize()
        index_ms = e0.elapsed_time(e1)
        del U_, L_

    def search(q_, d_, w_, p_, k_, index_base=0, out=None, **kw):  # kw: query_block, exchange (N > 1)
        i_, d2, st_ = B.nn_search(q_, d_, w_, p_, k_, index_base=index_base, out=out, return_stats=True,
                                  prefilter=not args.no_prefilter, keogh_only=args.keogh_only,
                                  stream=not args.no_stream, db_env=db_env, **kw)
        last["st"] = st_
        return i_, d2

    from paper_0811_3301_b200.sharded import query_sharded_nn_search

    def step(stats=False):
        if qshard:
            query_sharded_nn_search(qs, db, cfg.w, cfg.p, k, search=search)
        else:
            sharded_nn_search(qs, db, lo, cfg.w, cfg.p, k, search=search, merge=B.nn_merge, out_local=(idx, dst),
                              gather_bufs=gbufs, comm=comm)
        return last["st"] if stats else None

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step()
    barrier()
    stats_all = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gc.collect()
    gc.disable()  # no collector pause inside the timed region (the walk is host-driven)
    with ClockSampler(dev.index) as clk:
        time.sleep(0.5)  # let nvidia-smi start polling before the timed region (its start-up stalls the GPU)
        barrier()
        ev0.record(st)
        step_ev = []
        for _ in range(args.steps):
            stats_all.append(step(stats=True))
            step_ev.append(torch.cuda.Event(enable_timing=True))
            step_ev[-1].record(st)
        ev1.record(st)
        barrier()
    gc.enable()
    ms = ev0.elapsed_time(ev1) / args.steps
    # per-step device times (run-to-run diagnostics: one slow step shows up here)
    step_ms = [round((step_ev[i - 1] if i else ev0).elapsed_time(step_ev[i]), 3) for i in range(args.steps)]
    ms_t = torch.tensor([ms], device=dev)
    if ws > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())

    # ---- e2e: host (pinned) buffers through the same public call, copies inside the timed region ----
    qs_pin = torch.from_numpy(qs_h).pin_memory()
    db_pin = torch.from_numpy(db_h).pin_memory()
    h_idx = torch.empty((cfg.Q, k), dtype=torch.int64).pin_memory()
    h_dst = torch.empty((cfg.Q, k), dtype=torch.float32).pin_memory()
    e2e_steps = max(1, min(args.steps, 3))
    q_dev = torch.empty_like(qs)
    d_dev = torch.empty_like(db)

    def e2e_step():
        if ws == 1:  # the C-ABI host-pointer path: the library stages H2D / D2H itself
            B.nn_search(qs_pin, db_pin, cfg.w, cfg.p, k, index_base=lo, out=(h_idx, h_dst),
                        prefilter=not args.no_prefilter, keogh_only=args.keogh_only, stream=not args.no_stream)
        else:  # H2D of the shard + queries, sharded search (exchange, all-gather, merge), D2H
            q_dev.copy_(qs_pin, non_blocking=True)
            d_dev.copy_(db_pin, non_blocking=True)
            if qshard:
                gi, gd = query_sharded_nn_search(q_dev, d_dev, cfg.w, cfg.p, k, search=search)
            else:
                gi, gd = sharded_nn_search(q_dev, d_dev, lo, cfg.w, cfg.p, k, search=search, merge=B.nn_merge,
                                           out_local=(idx, dst), gather_bufs=gbufs, comm=comm)
            h_idx.copy_(gi, non_blocking=True)
            h_dst.copy_(gd, non_blocking=True)

    e2e_step()
    barrier()
    ev0.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    ev1.record(st)
    barrier()
    e2e_ms = torch.tensor([ev0.elapsed_time(ev1) / e2e_steps], device=dev)
    if ws > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # ---- work efficiency (after the timed region, 1 GPU): the cascade's LB_Improved and DTW
    # evaluations per query against their order-independent minima on a query sample, from the
    # library's own dense bounds and this run's final k-th distances tau_q: #{LB_Keogh <= tau(1+eps)}
    # (every such pair must reach LB_Improved) and #{LB_Improved <= tau(1+eps)} (must reach DTW)
    work_eff = None
    if ws == 1 and not args.keogh_only and not qshard:
        try:
            S = min(cfg.Q, 64)
            rows = torch.linspace(0, cfg.Q - 1, S).round().long().to(dev)
            qsamp = qs.index_select(0, rows).contiguous()
            U_, L_ = B.lb_envelope(qsamp, cfg.w)
            env_ = torch.stack([U_, L_]).contiguous()
            tau = dst.index_select(0, rows)[:, k - 1:k].double() * (1.0 + 1e-3) ** (1.0 / cfg.p)
            kb = B.lb_keogh(env_, db, cfg.p)
            n_keogh = int((kb.double() <= tau).sum().item())
            del kb
            ib = B.lb_improved(qsamp, env_, db, cfg.w, cfg.p)
            n_imp = int((ib.double() <= tau).sum().item())
            del ib
            st1 = stats_all[-1]
            work_eff = {"sample_queries": S,
                        "min_improved_per_query": n_keogh / S, "min_dtw_per_query": n_imp / S,
                        "improved_per_query": st1["improved_evaluated"] / cfg.Q,
                        "dtw_per_query": st1["dtw_evaluated"] / cfg.Q,
                        "improved_ratio": (st1["improved_evaluated"] / cfg.Q) / max(n_keogh / S, 1e-9),
                        "dtw_ratio": (st1["dtw_evaluated"] / cfg.Q) / max(n_imp / S, 1e-9)}
        except Exception as e:  # (a reporting extra: never fails the bench)
            work_eff = {"error": repr(e)[:200]}

    # ---- aggregate counters over ranks ----
    def tot(key):
        v = torch.tensor([float(sum(s[key] for s in stats_all) / len(stats_all))], device=dev,
                         dtype=torch.float64)
        if ws > 1:
            dist.all_reduce(v)
        return float(v.item())

    def max_ms(key):
        v = torch.tensor([statistics.mean(s[key] for s in stats_all)], device=dev)
        if ws > 1:
            dist.all_reduce(v, op=dist.ReduceOp.MAX)
        return float(v.item())

    keogh_ms = max_ms("ms_keogh")          # dense gate pass (piecewise-sum bound or LB_Keogh)
    surv_ms = max_ms("ms_survivor_kernel")  # survivor kernel (LB_Keogh + LB_Improved on sparse pairs)
    dtw_kernel_ms = max_ms("ms_dtw_kernel")  # banded-DTW kernel launches of the walk
    pairs = cfg.Q * cfg.N
    improved = tot("improved_evaluated")
    keogh_eval = tot("keogh_evaluated")
    dtw_eval = tot("dtw_evaluated")
    dtw_ab = tot("dtw_abandoned")
    cells_nom = tot("dtw_cells_nominal")
    cells_cmp = tot("dtw_cells_computed")
    launches = int(round(statistics.mean(s["kernel_launches"] for s in stats_all)))
    if rank == 0:
        pk = _peaks()
        sm_clock = 1965.0 if not pk else float(pk.get("sm_max_mhz", 1965.0))
        hbm_peak = 6533.5 if not pk else float(pk.get("hbm_gbs", 6533.5))
        n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
        # ALU issue peak: SMs x 4 schedulers x 32 lanes (one warp-instruction per scheduler per
        # clock = 128 lane-slots per SM per clock) x the max SM clock (guide unit counts)
        peak = n_sm * 128 * sm_clock * 1e6 / 1e12
        pairs_rank = cfg.Q * cfg.N / ws  # (query, candidate) pairs per rank, either sharding
        kern = {}
        # Minimal algorithmic issue slots per unit (sm_100a SASS):
        #  bound element (LB_Keogh, piecewise-sum): FADD2 (two elements' two subtractions, so 1 per
        #    element), FMNMX3 (max with 0), FFMA|FADD (accumulate)                   = 3
        #  LB_Improved element: FMNMX, FMNMX (envelope of H), FADD2 (1), FMNMX3, FFMA  = 5
        #  DTW cell (in the band |i-j| <= w, 0 <= j < n): FADD (x - y), FMNMX3, FADD|FFMA = 3
        if stream_mode:
            # HBM-bound: the database read once + beta1 written, per launch (one launch per step)
            bytes_ = cfg.N * cfg.n * 4 + cfg.Q * cfg.N * 4 + 2 * cfg.Q * cfg.n * 4
            kern["bound_pass"] = {"kernel": "keogh_stream_kernel (LB_Keogh, TMA-streamed database)",
                                  "bound": "hbm", "ms": keogh_ms, "work": bytes_ / 1e9, "unit": "GB/s",
                                  "peak": hbm_peak, "launches": 1,
                                  "note": "N*n*4 database bytes + Q*N*4 bound bytes per launch"}
        else:
            elems = 2 * (((cfg.n + 7) // 8 + 3) // 4 * 4) if pf else cfg.n
            kern["bound_pass"] = {"kernel": ("gate_sym_kernel (symmetric piecewise-sum gate, forward + reverse "
                                             "in one pass)" if pf else "keogh_tile_kernel (LB_Keogh)"),
                                  "bound": "alu", "ms": keogh_ms, "work": 3.0 * pairs_rank * elems / 1e12,
                                  "unit": "Tlane-op/s", "peak": peak, "launches": 1,
                                  "note": f"3 slots per pair-element, {elems} elements per pair"}
        if surv_ms > 0:
            k_in_kernel = keogh_eval if pf else 0.0
            kern["survivor_kernel"] = {"kernel": "improved_kernel (LB_Keogh + LB_Improved on sparse pairs)",
                                       "bound": "alu", "ms": surv_ms,
                                       "work": (3.0 * k_in_kernel + 5.0 * improved) * cfg.n / 1e12,
                                       "unit": "Tlane-op/s", "peak": peak,
                                       "note": "3n slots per LB_Keogh + 5n per LB_Improved evaluation (kernel counters)"}
            # its binding resource is the L1 / shared-memory data path (128 B/clk/SM, guide): the staged
            # candidate rows are read once per pair (x: 4n bytes per LB_Keogh, U(x), L(x): 8n per
            # LB_Improved) and the query rows once per (query, tile) entry (U, L, y, U(L), L(U): 20n)
            entries = tot("survivor_entries")
            l1_bytes = (4.0 * k_in_kernel + 8.0 * improved + 20.0 * entries) * cfg.n
            kern["survivor_kernel_l1"] = {"kernel": "improved_kernel (L1 / shared-memory bytes)", "bound": "smem",
                                          "ms": surv_ms, "work": l1_bytes / 1e9, "unit": "GB/s",
                                          "peak": n_sm * 128 * sm_clock * 1e6 / 1e9,
                                          "note": "4n B per LB_Keogh + 8n per LB_Improved + 20n per (query, tile) "
                                                  "entry through the SM's 128 B/clk data path",
                                          }
        if dtw_kernel_ms > 0:
            # w > 64: the four-lanes-per-pair kernel where it has an instantiation (csrc/dtw_wide.cu
            # wide_plan: band segments of 51 cells, w in {100, 101}; or unconstrained with n <= 256)
            wide = cfg.w > 64 and ((2 * cfg.w + 1 + 3) // 4 == 51 or (cfg.w >= cfg.n - 1 and cfg.n <= 256))
            kern["dtw_kernel"] = {"kernel": "dtw4_kernel (banded DTW walk)" if cfg.w <= 64 else
                                  ("dtw_wide_kernel (banded DTW walk, four lanes per pair)" if wide else
                                   "dtw_generic_kernel (banded DTW walk, w > 64)"),
                                  "bound": "alu", "ms": dtw_kernel_ms, "work": 3.0 * cells_cmp / 1e12,
                                  "unit": "Tlane-op/s", "peak": peak,
                                  "note": "3 slots per in-band DTW cell actually computed (kernel counter, early "
                                          "abandon), CUDA events around every walk-round launch"}
        # Measured instruction-mix peaks (scripts/isa_probe.cu, event-timed, profiles/r02h_isa_probe.txt,
        # profiles/r02x_isa_probe.txt for the midpoint-form gate element):
        # the same SASS sequences in 8 independent chains per thread, 32 warps per SM, elements (cells)
        # per SM clock.  FMNMX3 and the packed f32x2 ops issue at half rate and FFMA2 at a third, so a
        # bound element costs more than 3 issue slots: these are the kernels' attainable ALU roofs.
        mix = {"dtw_cell": 42.0, "lbk_elem": 26.0, "lbi_elem": 25.3, "gate_elem": 26.8, "lbk_packed": 27.7,
               "lb_pair": 24.6}  # lb_pair: FADD2 x2, FMNMX3 x2, FFMA x2 per element pair (streaming pass)
        clk_sm = n_sm * sm_clock * 1e6  # SM-clocks per second, whole GPU
        if "bound_pass" in kern and kern["bound_pass"]["bound"] == "alu":
            kern["bound_pass"]["mix_peak"] = 3.0 * mix["gate_elem"] * clk_sm / 1e12
        if "bound_pass" in kern and kern["bound_pass"]["bound"] == "hbm":
            # the LB_Keogh arithmetic caps the streaming pass too: Q pair-elements per database element
            rate = mix["lbk_packed"] if 4 < cfg.Q <= 8 else mix["lb_pair"]
            kern["bound_pass"]["alu_cap"] = rate * clk_sm / cfg.Q * 4 / 1e9  # GB/s of database
            kern["bound_pass"]["mix_peak"] = min(hbm_peak, kern["bound_pass"]["alu_cap"])
        if "survivor_kernel" in kern:
            kn = (keogh_eval if pf else 0.0) * cfg.n
            ki = improved * cfg.n
            t_mix = (kn / mix["lbk_elem"] + ki / mix["lbi_elem"]) / clk_sm
            kern["survivor_kernel"]["mix_peak"] = kern["survivor_kernel"]["work"] / t_mix if t_mix > 0 else peak
        if "dtw_kernel" in kern and cfg.w <= 64:
            kern["dtw_kernel"]["mix_peak"] = 3.0 * mix["dtw_cell"] * clk_sm / 1e12
        for v in kern.values():
            v["achieved"] = v["work"] / (v["ms"] * 1e-3) if v["ms"] > 0 else 0.0
            v["frac"] = v["achieved"] / v["peak"]
            if "mix_peak" in v:
                v["frac_of_mix_peak"] = v["achieved"] / v["mix_peak"]
        # SURVEY 8(d) "achieved fraction": the ideal step at the measured prune rates (each pass's
        # algorithmic work at its roofline, the hot passes only) over the measured step
        hot = [kk for kk in ("bound_pass", "survivor_kernel", "dtw_kernel") if kk in kern]
        ideal_peak = sum(kern[kk]["work"] / kern[kk]["peak"] for kk in hot) * 1e3
        ideal_mix = sum(kern[kk]["work"] / kern[kk].get("mix_peak", kern[kk]["peak"]) for kk in hot) * 1e3
        achieved_fraction = {"ideal_ms_at_peak": ideal_peak, "ideal_ms_at_mix_peak": ideal_mix,
                             "fraction_at_peak": ideal_peak / ms_max, "fraction_at_mix_peak": ideal_mix / ms_max,
                             "note": "sum over the bound pass, the survivor kernel and the DTW kernel of their "
                                     "algorithmic work (this step's measured prune rates) at the nominal / "
                                     "measured instruction-mix peak, divided by the measured step time"}
        dom_name = max((kk for kk in kern if kk != "survivor_kernel_l1"),
                       key=lambda kk: kern[kk]["ms"] / kern[kk].get("launches", 1))
        rk = kern[dom_name]
        traffic, traffic_note = None, None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            try:
                t = json.load(open(tpath)).get(f"{cfg.name}:{rk['kernel'].split()[0]}")
                if t:
                    traffic = t["bytes"]
                    traffic_note = t["note"]
            except Exception:
                traffic = None
        clocks = clk.summary()
        line = {
            "metric": "query-candidate pairs/s (exact DTW k-NN)",
            "value": pairs / (ms_max * 1e-3),
            "unit": "pairs/s",
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg.name, "Q": cfg.Q, "N": cfg.N, "n": cfg.n, "w": cfg.w, "p": cfg.p,
                       "k": cfg.k, "family": cfg.family,
                       "parallelism": f"query-shard{ws}" if qshard else f"db-shard{ws}",
                       "mode": ("stream" if stream_mode else ("prefilter" if pf else "alg3")) +
                               ("+keogh_only" if args.keogh_only else ""),
                       "db_index": ({"prebuilt": True, "build_ms": index_ms} if args.db_index else None),
                       "l2": f"inputs larger than L2 ({cfg.N * cfg.n * 4 / 1e9:.2f} GB database)"},
            "dtw_cells_per_s": cells_cmp / (ms_max * 1e-3),
            "dtw_cells_nominal_per_s": cells_nom / (ms_max * 1e-3),
            "dtw_kernel_cells_per_s": ({"computed": cells_cmp / (dtw_kernel_ms * 1e-3),
                                        "nominal": cells_nom / (dtw_kernel_ms * 1e-3)}
                                       if dtw_kernel_ms > 0 else None),
            "walk": {k2: statistics.mean(s[k2] for s in stats_all)
                     for k2 in ("range1_improved", "range1_dtw", "range1_cells", "walk_rounds", "dtw_evaluated",
                                "dtw_cells_computed")},
            "prune": {"prefilter": pf, "stream_mode": stream_mode, "keogh_only": bool(args.keogh_only),
                      "keogh_evaluated_frac": keogh_eval / pairs,
                      "keogh_pruned_frac": 1 - improved / pairs,
                      "improved_evaluated_frac": improved / pairs,
                      "dtw_evaluated_frac": dtw_eval / pairs,
                      "dtw_abandoned_frac_of_evaluated": dtw_ab / max(1.0, dtw_eval)},
            "stage_ms": {k2: statistics.mean(s[k2] for s in stats_all)
                         for k2 in ("ms_envelope", "ms_keogh", "ms_select", "ms_improved", "ms_survivor_kernel", "ms_dtw_kernel",
                                    "ms_dtw", "ms_total")},
            "roofline": {"kernel": rk["kernel"], "bound": rk["bound"], "achieved": rk["achieved"],
                         "peak": rk["peak"], "unit": rk["unit"], "frac": rk["frac"], "traffic": traffic,
                         "peak_note": (f"{n_sm} SMs x 128 lane-slots/clk x {sm_clock:.0f} MHz (guide unit counts, "
                                       "MEASURED_PEAKS sm_max_mhz)" if rk["bound"] == "alu" else
                                       "MEASURED_PEAKS hbm_gbs (measured copy bandwidth)"),
                         "ops_note": rk["note"], "kernel_ms": rk["ms"], "traffic_note": traffic_note,
                         "dominant": dom_name,
                         "mix_peak": rk.get("mix_peak"), "frac_of_mix_peak": rk.get("frac_of_mix_peak"),
                         "mix_note": "attainable peak of the kernel's own instruction mix, measured by "
                                     "scripts/isa_probe.cu (profiles/r02h_isa_probe.txt)",
                         **{kn: {x: v[x] for x in ("kernel", "bound", "ms", "achieved", "peak", "unit", "frac",
                                                   "mix_peak", "frac_of_mix_peak", "alu_cap") if x in v}
                            for kn, v in kern.items()}},
            "e2e": {"value": pairs / (e2e_ms * 1e-3), "unit": "pairs/s",
                    # whole job: every rank copies the queries and its shard in, its result out
                    "h2d_bytes_per_step": int(qs_h.nbytes * ws + cfg.N * cfg.n * 4 * (ws if qshard else 1)),
                    "d2h_bytes_per_step": int(cfg.Q * k * 12 * ws)},
            "work_efficiency": work_eff,
            "achieved_fraction": achieved_fraction,
            "gpu_launches": launches * args.steps + (0 if ws == 1 else args.steps),
            "clocks": clocks,
            "step_ms": step_ms,
        }
        if ws == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = oracle_sample(cfg, qs_h, db_h, budget_s=args.cpu_budget)
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--keogh-only", action="store_true",
                    help="Alg. 2 (LB_Keogh then DTW, no LB_Improved pass): the paper's comparison point")
    ap.add_argument("--shard", default="db", choices=["db", "queries"],
                    help="N > 1: shard the database (default, SURVEY 8(e)) or the queries (comparison "
                         "mode: replicated database, no collective during the search)")
    ap.add_argument("--py-exchange", action="store_true",
                    help="N > 1, database-sharded: threshold exchange by a Python torch.distributed callback "
                         "instead of the library's NCCL communicator")
    ap.add_argument("--no-stream", action="store_true",
                    help="Q <= 8: the tiled bound pass instead of the streaming one (DTWLB_NO_STREAM)")
    ap.add_argument("--db-index", action="store_true",
                    help="build the database index (row envelopes, nn_opts.db_env) once before the timed "
                         "region and reuse it in every step")
    ap.add_argument("--no-prefilter", action="store_true",
                    help="LB_Keogh over every pair (Alg. 3 as printed) instead of the piecewise-sum pre-filter")
    ap.add_argument("--w", type=int, default=None,
                    help="override the config's band w (the paper's w sweep, P:832-856); the workload "
                         "name gets a -w<w> suffix")
    args = ap.parse_args()
    cfg = datagen.CONFIGS[args.config]
    if args.w is not None and args.w != cfg.w:
        import dataclasses
        cfg = dataclasses.replace(cfg, w=args.w, name=f"{cfg.name}-w{args.w}")
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
