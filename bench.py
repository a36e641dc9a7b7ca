#!/usr/bin/env python
"""Benchmark: exact assignment solves/s on BASELINE config 3 (4096 independent
n=128 instances, instances sharded across GPUs), plus the reference's CPU
solver timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

A step = one batched solve of this rank's shard of the 4096 instances
(strong scaling: the job total is fixed).  ``value`` = 4096 / (max over ranks
of the mean device time per step) with inputs resident in HBM, through the
stream-ordered call kmb_solve_batch_async_i32 (statuses checked after the timed
region; the synchronous kmb_solve_batch_i32 is reported beside it as
``sync_call``); ``e2e`` is the same through the synchronous C ABI call with
pinned HOST buffers (H2D of the costs and D2H of assignment + duals + totals
inside the timed region).  L2 is flushed (a
256 MiB write) before every timed step.  At N=1, rank 0 also runs the
config-5 (n=16384, 1 GiB) single-instance solve, whose reduced-cost scan is the
HBM-bound kernel, and reports its roofline under ``extras`` (disable with
--no-extras).  Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
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

METRIC = "assignment solves/sec (and n×n cost GB/s streamed vs HBM peak) at 1/2/4/8 GPUs"
BATCH, N = 4096, 128
WORKLOAD = "c3: 4096 independent n=128 instances, 300-D N(0,1) fp32 vectors, llround(1e4*dist)"
FALLBACK_HBM = 6650.0


def peaks() -> tuple[float, str]:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region.  NVML is
    polled every ~2 ms from a thread (the timed regions last tens of ms, too short
    for nvidia-smi's ~100 ms per query); nvidia-smi is the fallback."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, float, tuple]] = []
        self.source = "nvidia-smi"
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(index)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            self._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            self._nvml = pynvml
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        nv = self._nvml
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        bits = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        return float(sm), float(mx), tuple(bool(r & b) for b in bits)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5)
        if out.returncode != 0 or not out.stdout.strip():
            return None
        s = [x.strip() for x in out.stdout.strip().split(",")]
        return float(s[0]), float(s[1]), tuple(x.lower() == "active" for x in s[2:6])

    def _run(self):
        while True:
            try:
                smp = self._sample_nvml() if self._nvml else self._sample_smi()
                if smp:
                    self.samples.append(smp)
            except Exception:
                pass
            if self._stop.wait(0.002 if self._nvml else 0.2):
                break

    def __enter__(self):  # re-enterable: samples of every region accumulate
        self._stop.clear()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted({self.NAMES[k] for s in self.samples for k in range(4) if s[2][k]})
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples), "reasons": reasons,
                "samples": len(self.samples), "source": self.source}


_BACKEND = "gloo"


def dist_setup(args):
    """One process per GPU (torchrun).  NCCL carries the barrier and the
    max-over-ranks reduction; when ranks outnumber visible GPUs (a 1-GPU box
    exercising the multi-rank path) ranks share devices and gloo is used, since
    NCCL refuses two ranks on one device."""
    global _BACKEND
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    device = local
    if world > 1:
        import torch
        import torch.distributed as dist
        ndev = torch.cuda.device_count() if args.impl == "ours" else 0
        if args.impl == "ours" and ndev >= int(os.environ.get("LOCAL_WORLD_SIZE", world)):
            _BACKEND = "nccl"
            torch.cuda.set_device(local)
        else:
            _BACKEND = "gloo"
            if ndev:
                device = local % ndev
        dist.init_process_group(_BACKEND)
    return world, rank, device


def shard(world: int, rank: int) -> tuple[int, int]:
    per = BATCH // world
    extra = BATCH % world
    first = rank * per + min(rank, extra)
    return first, per + (1 if rank < extra else 0)


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda" if _BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def cpu_reference_rate(costs: np.ndarray, seconds: float, threads: int) -> tuple[float, int, float]:
    """Reference solve_batched_km (lossless B, oracle/_ref) on `threads` host
    threads over chunks of `costs` until ~`seconds` of wall time; returns
    (solves/s, instances solved, wall seconds)."""
    import oracle as O
    done, wall = 0, 0.0
    chunk = max(threads * 8, 32)
    while wall < seconds and done < costs.shape[0]:
        part = costs[done: done + chunk]
        _, w = O.ref_solve_many_i32(part, mode=1, nthreads=threads)
        done += part.shape[0]
        wall += w
    return done / wall, done, wall


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU solver on the box's host cores."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    first, count = 0, args.ref_sample
    costs = _gen_c3(first, count)
    import oracle as O
    rates = []
    for s in range(args.warmup + args.steps):
        _, w = O.ref_solve_many_i32(costs, mode=1, nthreads=threads)
        if s >= args.warmup:
            rates.append(count / w)
    value = statistics.mean(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * count / value, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded, BASELINE config 3 shapes)",
        "config": {"workload": WORKLOAD, "batch": BATCH, "n": N,
                   "sample_per_step": count, "solver": "ot::solve_batched_km, B = N (lossless)"},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": "reference",
                         "sample": f"{count} of the 4096 config-3 instances per step, "
                                   f"unmodified reference (oracle/_ref), {threads} threads"},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _gen_c3(first: int, count: int) -> np.ndarray:
    from paper_2005_01182_b200 import workloads as W
    return W.embedding_batch(count, N, 300, 1e4, seed=3, first=first)


# engine id (kmb_stats.engine) -> (description, kernel); the auto choice depends on
# the per-GPU shard: all 4096 instances at 1-2 GPUs run one warp each, the 1024 /
# 512-instance shards at 4 / 8 GPUs one CTA each
ENGINES = {4: ("warp engine (one warp per instance, costs streamed from L2)", "k_warp_batch"),
           6: ("CTA engine (one CTA per instance, thread per column, costs from L2)", "k_cta_batch"),
           3: ("warp engine, matrices staged in SMEM by TMA", "k_warp_batch"),
           2: ("CTA engine, matrices staged in SMEM by TMA", "k_cta_batch")}


def extras_c5(solver, hbm_peak: float) -> dict:
    """Config 5 (n=16384, 1 GiB, HBM-resident): one warm + timed solves, the
    reduced-cost scan's algorithmic bytes over the device time."""
    import torch
    from paper_2005_01182_b200 import workloads as W
    c = W.CONFIGS["c5"].make()
    n = c.shape[0]
    dc = torch.from_numpy(c).cuda()
    r2c = torch.empty(n, dtype=torch.int32, device="cuda")
    u = torch.empty(n, dtype=torch.int64, device="cuda")
    v = torch.empty(n, dtype=torch.int64, device="cuda")
    tot = torch.empty(1, dtype=torch.int64, device="cuda")
    times, st = [], None
    for it in range(3):
        st = solver.solve_into(dc, n, n, 1, r2c, u, v, tot)
        if it:
            times.append(st.seconds)
    t = statistics.mean(times)
    # bytes the engine's scans read: full rows + dirty-segment re-relaxes (16 B
    # per row-segment) + the two reductions
    rd = 4.0 * n * (st.rows_scanned + 2 * n) + 16.0 * st.segment_rows
    # SURVEY 8(d)2 solve-level effective rate: one 4n^2 pass per phase + 2 reductions
    eff = 4.0 * n * n * (st.phases + 2)
    return {"workload": "c5: n=16384 U{0..1e6}, 1 GiB int32, single GPU",
            "solve_ms": 1e3 * t, "solves_per_s": 1.0 / t, "phases": st.phases,
            "dual_steps": st.dual_steps, "rows_scanned": st.rows_scanned,
            "scan_roofline": {"bound": "hbm", "achieved": eff / t / 1e9, "peak": hbm_peak,
                              "unit": "GB/s", "frac": eff / t / 1e9 / hbm_peak,
                              "note": "SURVEY 8(d)2 effective rate 4*n^2*(phases+2)/solve time "
                                      "(the reference's one-pass-per-phase work)"},
            "bytes_read_gbs": rd / t / 1e9,
            "bytes_read_note": "what the scans actually read: 4*n*(rows_scanned+2n) + "
                               "16*segment_rows (epoch-start re-relaxes touch dirty segments only)",
            "segment_rows": st.segment_rows}


def extras_single(solver) -> dict:
    """Configs 1, 2 and 4 (single instances, device-resident): best of 3 solves
    on the auto-selected engine, total cost checked against the committed golden."""
    import torch
    from paper_2005_01182_b200 import workloads as W
    names = {6: "CTA", 8: "single-CTA (512 threads)", 5: "cluster (DSMEM state)", 1: "grid"}
    golden = {}
    gp = os.path.join(ROOT, "tests", "golden", "configs.json")
    if os.path.exists(gp):
        with open(gp) as f:
            golden = json.load(f)
    out = {}
    for key in ("c1", "c2", "c4"):
        c = W.CONFIGS[key].make()
        n = c.shape[0]
        dc = torch.from_numpy(c).cuda()
        r2c = torch.empty(n, dtype=torch.int32, device="cuda")
        u = torch.empty(n, dtype=torch.int64, device="cuda")
        v = torch.empty(n, dtype=torch.int64, device="cuda")
        tot = torch.empty(1, dtype=torch.int64, device="cuda")
        best, st = None, None
        for _ in range(3):
            st = solver.solve_into(dc, n, n, 1, r2c, u, v, tot)
            best = st.seconds if best is None else min(best, st.seconds)
        g = golden.get(key, {})
        ok = None
        if "total_cost" in g and "u_fnv" in g and "v_fnv" in g:  # reference's cost and duals
            ok = (int(tot[0]) == int(g["total_cost"])
                  and W.fnv1a64(u.cpu().numpy()) == g["u_fnv"] and W.fnv1a64(v.cpu().numpy()) == g["v_fnv"])
        out[key] = {"n": n, "solve_ms": 1e3 * best, "engine": names.get(st.engine, str(st.engine)),
                    "rounds": st.rounds, "total_cost": int(tot[0]), "matches_reference_golden": ok}
    return out


def extras_auction(solver) -> dict:
    """Config-3 batch through the GPU auction (ot::solve_auction_scaled, exact
    schedule; device-resident costs), and the unmodified reference auction on
    one host thread over a bounded sample of the same instances."""
    import time
    import torch
    import oracle as O
    from paper_2005_01182_b200 import workloads as W
    from paper_2005_01182_b200.api import AuctionConfig
    c = W.CONFIGS["c3"].make()
    b, n, _ = c.shape
    dc = torch.from_numpy(c).cuda()
    pr = torch.empty((b, n), dtype=torch.float64, device="cuda")
    r2c = torch.empty((b, n), dtype=torch.int32, device="cuda")
    tot = torch.empty(b, dtype=torch.int64, device="cuda")
    bids = torch.empty(b, dtype=torch.int64, device="cuda")
    cfg = AuctionConfig(1, 0.0, 4.0, 0.0, 10**9, 0.0)
    t = min(solver.auction_into(dc, b, n, cfg, pr, r2c, tot, bids) for _ in range(3))
    k, t0 = 32, time.perf_counter()
    for i in range(k):
        r = O.ref_solve_auction_scaled(c[i])
        if r.iterations != int(bids[i]) or r.total_cost != int(tot[i]):
            raise RuntimeError(f"auction mismatch on instance {i}")
    ref = k / (time.perf_counter() - t0)
    return {"workload": "c3 through solve_auction_scaled (exact schedule), 4096 x n=128",
            "gpu_ms": 1e3 * t, "solves_per_s": b / t, "bids_mean": float(bids.double().mean()),
            "reference_solves_per_s_1_thread": ref,
            "reference_sample": f"first {k} instances, unmodified reference auction, 1 thread; "
                                "bids and totals checked equal"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--ref-sample", type=int, default=1024)
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        return

    import torch
    from paper_2005_01182_b200 import Solver
    torch.cuda.set_device(local)
    first, count = shard(world, rank)
    host = _gen_c3(first, count)
    solver = Solver(local)
    stream = torch.cuda.current_stream()
    solver.set_stream(stream.cuda_stream)

    dev = torch.device("cuda", local)
    dcost = torch.from_numpy(host).to(dev)
    r2c = torch.empty((count, N), dtype=torch.int32, device=dev)
    du = torch.empty((count, N), dtype=torch.int64, device=dev)
    dv = torch.empty((count, N), dtype=torch.int64, device=dev)
    dtot = torch.empty(count, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)

    # pinned host buffers for the end-to-end leg
    hcost = torch.from_numpy(host).pin_memory()
    hr2c = torch.empty((count, N), dtype=torch.int32).pin_memory()
    hu = torch.empty((count, N), dtype=torch.int64).pin_memory()
    hv = torch.empty((count, N), dtype=torch.int64).pin_memory()
    htot = torch.empty(count, dtype=torch.int64).pin_memory()

    dstatus = torch.full((count,), -1, dtype=torch.int32, device=dev)
    phases = 0
    engine_used = 4
    for _ in range(args.warmup):
        st = solver.solve_batch_into(dcost, count, N, 1, r2c, du, dv, dtot)
        phases = st.phases
        engine_used = st.engine
        solver.solve_batch_async(dcost, count, N, 1, r2c, du, dv, dtot, dstatus)
    torch.cuda.synchronize()

    def timed_steps(call) -> float:
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        barrier(world)
        torch.cuda.synchronize()
        with clk:
            for k in range(args.steps):
                flush.fill_(k)
                ev[k][0].record(stream)
                call()
                ev[k][1].record(stream)
            torch.cuda.synchronize()
        barrier(world)
        return statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev)

    clk = ClockSampler(local)
    # value: the stream-ordered call (kmb_solve_batch_async_i32), one batch per
    # step, statuses checked after the timed region
    dstatus.fill_(-1)
    step_ms = timed_steps(lambda: solver.solve_batch_async(dcost, count, N, 1, r2c, du, dv, dtot, dstatus))
    if int(dstatus.abs().sum()) != 0:
        raise RuntimeError("bench: an instance reported a nonzero status")
    step_ms_max = max_over_ranks(step_ms, world)
    value = BATCH / (step_ms_max * 1e-3)
    # the synchronous call (status fold + host wait per step), reported beside it
    sync_ms = max_over_ranks(timed_steps(lambda: solver.solve_batch_into(dcost, count, N, 1, r2c, du, dv, dtot)), world)

    # end to end through the C ABI with host buffers (H2D + kernel + D2H)
    for _ in range(max(1, args.warmup)):
        solver.solve_batch_into(hcost, count, N, 1, hr2c, hu, hv, htot, stats=False)
    e2e_ms = max_over_ranks(timed_steps(
        lambda: solver.solve_batch_into(hcost, count, N, 1, hr2c, hu, hv, htot, stats=False)), world)
    ok_e2e = bool(torch.equal(hr2c, r2c.cpu())) and bool(torch.equal(htot, dtot.cpu()))

    hbm_peak, peak_src = peaks()
    # roofline of the dominant kernel (k_warp_batch): SURVEY.md §8(d) algorithmic
    # bytes = 4*n^2 per phase + 2*4*n^2 for the reductions, per instance
    alg_bytes = 4.0 * N * N * (phases + 2 * count)
    achieved = alg_bytes / (step_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_batch_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    extras = None
    cpu = None
    if rank == 0 and world == 1:
        if not args.no_extras:
            extras = {}
            for key, fn in (("c5", lambda: extras_c5(solver, hbm_peak)),
                            ("single_instances", lambda: extras_single(solver)),
                            ("auction_c3", lambda: extras_auction(solver))):
                try:
                    extras[key] = fn()
                except Exception as e:  # reported, never silently dropped
                    extras[key] = {"error": repr(e)}
                # hand the freed 1 GiB c5 segment back: a later matrix carved out
                # of torch's cached segment solved ~10% slower (c4: 129 vs 142 ms,
                # tools/ex_probe.py), an address-placement effect of the harness
                torch.cuda.empty_cache()
        threads = os.cpu_count() or 1
        try:
            rate, done, wall = cpu_reference_rate(host, args.cpu_seconds, threads)
            cpu = {"value": rate, "unit": "solves/s", "cores": threads, "kind": "reference",
                   "sample": f"first {done} config-3 instances, unmodified reference "
                             f"solve_batched_km (oracle/_ref, lossless B) on {threads} threads, "
                             f"{wall:.1f} s"}
        except Exception as e:
            cpu = {"value": None, "unit": "solves/s", "cores": threads, "kind": "reference",
                   "sample": f"unavailable: {e!r}"}

    # the ncu DRAM bytes were captured on the 4096-instance warp-engine launch
    traffic_used = traffic if (engine_used == 4 and count == BATCH) else None
    dram_gbs = traffic_used / (step_ms * 1e-3) / 1e9 if traffic_used else None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic (seeded, BASELINE config 3 shapes)",
            "config": {"workload": WORKLOAD, "batch": BATCH, "n": N, "per_rank": count,
                       "parallelism": f"instances sharded over {world} rank(s), one per GPU "
                                      f"({_BACKEND} for the max-over-ranks timing)",
                       "l2": "flushed (256 MiB write) before every timed step",
                       "api": "value: kmb_solve_batch_async_i32 (stream-ordered, device buffers, "
                              "statuses checked after the timed region); e2e: kmb_solve_batch_i32 "
                              "with pinned host buffers",
                       "engine": ENGINES.get(engine_used, (str(engine_used), ""))[0]},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic_used,
                         "kernel": ENGINES.get(engine_used, ("", "?"))[1], "peak_source": peak_src,
                         "dram_gbs": dram_gbs, "dram_frac": (dram_gbs / hbm_peak) if dram_gbs else None,
                         "note": "L1/L2-resident re-reads: algorithmic bytes are SURVEY 8(d)'s "
                                 "4n^2 per phase (+2 reductions) per instance, mostly served from "
                                 "L2, so achieved can exceed the HBM peak; traffic = ncu DRAM "
                                 "bytes of one launch of this kernel on this shard "
                                 "(profiles/ncu_batch_summary.json), dram_gbs = traffic / the "
                                 "live per-launch time: the HBM view of the same launch"},
            "cpu_baseline": cpu,
            "e2e": {"value": BATCH / (e2e_ms * 1e-3), "unit": "solves/s",
                    "h2d_bytes_per_step": int(host.nbytes),
                    "d2h_bytes_per_step": int(count * N * (4 + 8 + 8) + count * 8 + count * 4),
                    "matches_device_run": ok_e2e},
            # per timed step of the value leg (the stream-ordered call): the
            # engine kernel — profiles/r01_bench_launches.csv
            "gpu_launches": args.steps,
            "sync_call": {"api": "kmb_solve_batch_i32 (status fold + host wait per step)",
                          "ms_per_step": sync_ms, "value": BATCH / (sync_ms * 1e-3)},
            "clocks": clk.summary(),
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
