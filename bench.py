#!/usr/bin/env python
"""Benchmark: time-to-min-cut and Mnodes/s on the 67M-node column graph (BASELINE.json
`metric`; config C4 = 512x512x256, Delta = 4).

One step = the whole hot path on one synthetic volume that is
already resident in HBM: colgraph_build -> maxflow_solve -> mincut_extract_surface.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]

N > 1 is launched by torchrun (one rank per GPU).  Rank 0 prints ONE JSON line.
`--impl reference` times the CPU oracle (oracle/, Dinic on the explicit graph) on a
bounded crop of the same workload on this box's host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import volumes as V  # noqa: E402

METRIC = "Mnodes/s and time-to-min-cut (s), 67M-node column graph"
UNIT = "Mnodes/s"
REF_CROP = 64      # --impl reference: x, y < REF_CROP crop (full Z) per step
BASE_CROP = 96     # cpu_baseline leg: x, y < BASE_CROP crop (full Z)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    return ap.parse_args()


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def workload_config(spec, extra=None):
    cfg = {"workload": f"{spec.name} {spec.X}x{spec.Y}x{spec.Z} Delta={spec.delta} ({spec.n:,} nodes)",
           "n_nodes": spec.n, "X": spec.X, "Y": spec.Y, "Z": spec.Z, "delta": spec.delta,
           "input_sha256": V.MANIFEST.get(spec.name),
           "l2": "inputs larger than L2 (32 B/node SoA = %.2f GiB vs 126 MB L2)" % (spec.n * 32 / 2**30)}
    if extra:
        cfg.update(extra)
    return cfg


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu capture, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return None
    return None


class ClockSampler:
    """nvidia-smi-equivalent clocks / throttle reasons sampled during the timed region (NVML)."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self.nv, self.err = None, str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.nv:
            return {"error": getattr(self, "err", "nvml unavailable")}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_oracle_rate(c_crop, delta):
    import oracle
    t = time.perf_counter()
    r = oracle.colgraph_solve(c_crop, delta, want_mask=False)
    dt = time.perf_counter() - t
    assert r["status"] == 0
    return c_crop.size / dt / 1e6, dt


def run_reference(args, spec):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    oracle.build()
    c = V.generate(spec)
    crop = np.ascontiguousarray(c[:REF_CROP, :REF_CROP, :])
    for _ in range(args.warmup):
        cpu_oracle_rate(crop, spec.delta)
    times = []
    for _ in range(args.steps):
        _, dt = cpu_oracle_rate(crop, spec.delta)
        times.append(dt)
    ms = 1000.0 * sum(times) / len(times)
    value = crop.size / (ms / 1000.0) / 1e6
    sample = f"{spec.name} crop x,y < {REF_CROP}, all z ({crop.size:,} nodes) per step; single-threaded Dinic"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": workload_config(spec, {"sample": sample}),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "time_to_min_cut_s_for_sample": ms / 1000.0, "host_cores": os.cpu_count()}
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, spec):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2601_17026_b200 import colgraph as cg
    from paper_2601_17026_b200 import dist as cgd
    stream = torch.cuda.current_stream(dev)
    X, Y, Z = spec.X, spec.Y, spec.Z
    # this rank's x-slab (N = 1: the whole volume), generated directly (same bytes as the slice)
    x0, x1 = cgd.slab(X, rank, world) if world > 1 else (0, X)
    c_host = V.generate(spec, x_range=(x0, x1))
    if world == 1:
        assert V.sha256_volume(c_host) == V.MANIFEST[spec.name], "synthetic input differs from the pinned manifest"
    c_pin = torch.from_numpy(c_host).pin_memory()
    cost = c_pin.to(dev, non_blocking=False)
    nccl_id = cgd.init_nccl_id() if world > 1 else None
    opts = cg.make_opts()
    surface = torch.empty((x1 - x0, Y), dtype=torch.int32, device=dev)

    def step(cost_dev):
        if world > 1:
            r = cgd.solve_slab(cost_dev, (X, Y, Z, spec.delta), rank, world, nccl_id, opts=opts, stream=stream)
            assert r["status"] == cg.CG_OK and r["extract_status"] == cg.CG_OK, (r["status"], r["extract_status"])
            return r["flow"], r["stats"], r["surface"]
        h = cg.colgraph_build(cost_dev, spec.delta, stream=stream)
        try:
            st, flow, _ = cg.maxflow_solve(h, opts)
            assert st == cg.CG_OK, cg.STATUS.get(st)
            est = cg.mincut_extract_surface(h, surface)
            assert est == cg.CG_OK, cg.STATUS.get(est)
            return flow, cg.colgraph_stats(h), surface
        finally:
            cg.colgraph_free(h)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(ms):
        if world == 1:
            return ms
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 0)):
        step(cost)
    barrier()
    stats = []
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        step_ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        ev0.record(stream)
        step_ev[0].record(stream)
        for k in range(args.steps):
            flow, s, surf_last = step(cost)
            s = dict(s, flow=flow)
            stats.append(s)
            step_ev[k + 1].record(stream)
        ev1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(ev0.elapsed_time(ev1))
    # every timed step's |f| and the last step's surface against the oracle's stored result
    # (tests/golden, written by scripts/make_oracle_golden.py from oracle/ only)
    golden_ok = None
    gpath = os.path.join(ROOT, "tests", "golden", f"oracle_{spec.name}.json")
    if os.path.exists(gpath):
        import hashlib
        gold = json.load(open(gpath))
        flows = {st["flow"] for st in stats}
        assert flows == {gold["flow"]}, (flows, gold["flow"])
        surf_all = cgd.gather_slabs(surf_last.cpu().numpy()) if world > 1 else surf_last.cpu().numpy()
        assert hashlib.sha256(surf_all.astype("<i4").tobytes()).hexdigest() == gold["surface_sha256"]
        golden_ok = True
    step_ms = sorted(step_ev[k].elapsed_time(step_ev[k + 1]) for k in range(args.steps))
    ms_step = ms_total / args.steps
    value = spec.n * args.steps / (ms_total / 1000.0) / 1e6  # whole volume per step, all ranks together

    # e2e through the public API: every step copies this rank's cost slab from pinned host
    # memory, solves, and reads the surface (+ |f|) back to the host
    e2e_steps = args.e2e_steps or args.steps
    cost_e2e = torch.empty_like(cost)
    surf_host = torch.empty((x1 - x0, Y), dtype=torch.int32).pin_memory()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        if world == 1:
            r = cg.colgraph_solve_host_ptr(c_pin, spec.delta, surf_host, stream=stream)
            assert r["status"] == 0 and r["flow"] == flow
        else:
            cost_e2e.copy_(c_pin, non_blocking=True)
            f2, _, surf_dev = step(cost_e2e)
            surf_host.copy_(surf_dev)
            assert f2 == flow
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1)) / e2e_steps
    e2e_value = spec.n / (e2e_ms / 1000.0) / 1e6

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return 0

    sweep_ms = sum(s["ms_sweep_kernels"] for s in stats)
    sweep_bytes = sum(s["sweep_bytes_alg"] for s in stats)
    sweeps = sum(s["sweeps"] for s in stats)
    peak, peak_src = measured_peak()
    achieved = sweep_bytes / (sweep_ms / 1000.0) / 1e9 if sweep_ms > 0 else 0.0
    tr = ncu_traffic()
    roofline = {"kernel": "push-relabel sweep (k_walk_ws / k_sweep_v)", "bound": "hbm", "achieved": achieved,
                "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_source": peak_src,
                "traffic": tr.get("sweep_dram_bytes_per_launch") if tr else None,
                # the ncu'd solve replays an unprofiled solve's relabel schedule (CG_GR_SCHEDULE);
                # its own algorithmic bytes per launch and the ratio are given beside the traffic
                "traffic_alg_bytes_per_launch": tr.get("sweep_alg_bytes_per_launch_same_run") if tr else None,
                "traffic_over_alg": tr.get("traffic_over_alg") if tr else None,
                "traffic_source": tr.get("source") if tr else None,
                "alg_bytes_per_launch": sweep_bytes / max(sweeps, 1),
                "avg_launch_us": 1000.0 * sweep_ms / max(sweeps, 1),
                "alg_bytes_def": "SURVEY.md §8(d): 32 B per vertex visit (state read) + 12 B per push + "
                                 "4 B per relabel",
                "relabel_share_of_ops": sum(s["relabel_ops"] for s in stats) / max(1, sum(s["work"] for s in stats)),
                "share_of_step": sweep_ms * args.steps / (ms_total * len(stats)) if ms_total > 0 else None}
    # global relabel (a2/a5): SURVEY.md §8(d) prices a full pass at 28 B per vertex (read T, D, L;
    # write H); achieved = that x n per relabel / the relabel's average wall time in the solve
    n_gr = sum(s["global_relabels"] for s in stats)
    gr_ms = sum(s["ms_global_relabel"] for s in stats)
    gr_alg = 28.0 * spec.n
    roofline_gr = {"kernel": "global relabel (exact reverse BFS / column fixpoint)", "bound": "hbm",
                   "achieved": gr_alg * n_gr / (gr_ms / 1000.0) / 1e9 if gr_ms > 0 else 0.0, "peak": peak,
                   "unit": "GB/s", "alg_bytes_per_relabel": gr_alg, "avg_relabel_ms": gr_ms / max(n_gr, 1),
                   "alg_bytes_def": "28 B per vertex per relabel (SURVEY.md §8(d))"}
    roofline_gr["frac"] = roofline_gr["achieved"] / peak
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "time_to_min_cut_s": ms_step / 1000.0,
            "ms_per_step_min_median_max": [step_ms[0], step_ms[len(step_ms) // 2], step_ms[-1]],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "int32", "data": "synthetic (seeded generator synth/volumes.py, sha256-pinned)",
            "config": workload_config(spec, {"parallelism": f"x-slab{world}" if world > 1 else "single-gpu"}),
            "flow": flow, "flow_matches_oracle_golden": golden_ok, "roofline": roofline, "roofline_relabel": roofline_gr,
            "e2e": {"value": e2e_value, "unit": UNIT, "ms_per_step": e2e_ms, "h2d_bytes_per_step": 4 * spec.n,
                    "d2h_bytes_per_step": 4 * X * Y + 8},
            "gpu_launches": int(sum(s["kernel_launches"] for s in stats)),
            "solver": {"sweeps_per_step": sweeps / len(stats),
                       "global_relabels_per_step": sum(s["global_relabels"] for s in stats) / len(stats),
                       "gr_passes_per_step": sum(s["gr_passes"] for s in stats) / len(stats),
                       "extract_passes_per_step": sum(s["extract_passes"] for s in stats) / len(stats),
                       "ms_sweep_kernels_per_step": sweep_ms / len(stats),
                       "ms_global_relabel_per_step": sum(s["ms_global_relabel"] for s in stats) / len(stats),
                       "ms_extract_per_step": sum(s["ms_extract"] for s in stats) / len(stats),
                       "ms_build_per_step": sum(s["ms_build"] for s in stats) / len(stats),
                       "work_per_step": sum(s["work"] for s in stats) / len(stats)},
            "clocks": clk.summary(), "library": cg.version()}
    if world == 1 and not args.no_cpu_baseline:
        crop = np.ascontiguousarray(c_host[:BASE_CROP, :BASE_CROP, :])
        rate, dt = cpu_oracle_rate(crop, spec.delta)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle",
                                "sample": f"{spec.name} crop x,y < {BASE_CROP}, all z ({crop.size:,} nodes), "
                                          f"single-threaded Dinic, {dt:.1f} s"}
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    args = parse()
    spec = V.CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, spec)
    return run_ours(args, spec)


if __name__ == "__main__":
    sys.exit(main())
