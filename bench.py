"""Benchmark: GRNND graph build at SIFT1M shape (1M x 128 fp32, L2) on B200.

BASELINE.json metric: "build seconds at 1M x 128 (1/2/4/8 B200); graph recall@10 vs
CPU ref".  Workload (configs[1]): synthetic gaussian 1,000,000 x 128
(generate(..., "gaussian", seed=1)), S=20 R=96 T1=4 T2=15 rho=0.6 seed=1, pair order
"disordered".  One step = one complete build (init + 60 update + 3 reverse rounds +
CSR finalize).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--n N] [--dim D]

value  : device-timed build seconds with the vectors already resident in HBM (CUDA events
         on the launching stream, barrier + synchronize on both sides, max over ranks).
e2e    : the same build through the public API paper_2510_02774_b200.build(Dataset) from
         pinned host memory -- H2D of the vectors and D2H of the CSR graph inside the
         timed region.
cpu_baseline / --impl reference: the CPU oracle (oracle/, a C port of the reference's
         numba kernels, all host threads) on a bounded sample of the same workload: init,
         the first 2 update rounds, 1 reverse round and finalize at full 1M x 128, with the
         remaining update rounds extrapolated by their reference-semantics pair counts.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "build seconds at 1M×128 (1/2/4/8 B200); graph recall@10 vs CPU ref"
WORKLOAD = "SIFT1M-shape synthetic 1M×128 fp32 L2, R=96, single B200"
PARAMS = dict(S=20, R=96, T1=4, T2=15, rho=0.6, seed=1)
PAIRS_FILE = ROOT / "profiles" / "c2_round_pairs.json"
NCU_FILE = ROOT / "profiles" / "r1f_pair_phase_ncu.json"
CPU_PROFILE = ROOT / "profiles" / "c2_cpu_rounds.json"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    return ap.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
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
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU leg
def round_pairs(T1: int, T2: int):
    """Reference-semantics pair evaluations per update round of this workload (a
    deterministic property of the build; recorded from the GPU run, whose graph is
    bit-identical to the reference's)."""
    try:
        d = json.loads(PAIRS_FILE.read_text())
        if d["n"] == 1_000_000 and len(d["pairs_ref"]) == T1 * T2:
            return d["pairs_ref"]
    except Exception:
        pass
    return None


def cpu_round_profile(n: int):
    try:
        d = json.loads(CPU_PROFILE.read_text())
        return d if d["n"] == n else None
    except Exception:
        return None


def cpu_sample(data: np.ndarray, pairs: list | None):
    """Bounded CPU sample (about 10-30 s): oracle init, 2 update rounds, 1 reverse round,
    finalize at full size on all host threads; returns (estimated build seconds, info)."""
    import oracle

    threads = oracle.max_threads()
    p = PARAMS
    n_up = p["T1"] * p["T2"]
    t0 = time.perf_counter()
    st = oracle.State(data, p["S"], p["R"], p["seed"])
    t_init = time.perf_counter() - t0
    t_up = []
    for r in range(2):
        t0 = time.perf_counter()
        st.update_round(p["seed"], 1 + r, 0)
        t_up.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    st.reverse_round(p["rho"])
    t_rev = time.perf_counter() - t0
    t0 = time.perf_counter()
    st.finalize()
    t_fin = time.perf_counter() - t0
    del st
    prof = cpu_round_profile(data.shape[0])
    if prof:
        # the measured per-round shape of one full CPU build of this workload on this
        # host type (profiles/c2_cpu_rounds.json): scale the sampled rounds by it
        up = [r["seconds"] for r in prof["rounds"] if r["kind"] == "update"]
        rv = [r["seconds"] for r in prof["rounds"] if r["kind"] == "reverse"]
        t_updates = sum(t_up) * sum(up) / (up[0] + up[1])
        t_revs = t_rev * sum(rv) / rv[0]
        how = (f"rounds extrapolated with the per-round shape of a measured full CPU build "
               f"({prof['total_s']:.1f}s, {prof['threads']} threads, profiles/c2_cpu_rounds.json)")
    elif pairs:
        per_pair = sum(t_up) / float(pairs[0] + pairs[1])
        t_updates = sum(t_up) + per_pair * float(sum(pairs[2:]))
        t_revs = (p["T1"] - 1) * t_rev
        how = "update rounds 3..60 extrapolated by reference-semantics pair counts"
    else:
        t_updates = sum(t_up) / 2 * n_up
        t_revs = (p["T1"] - 1) * t_rev
        how = "update rounds 3..60 extrapolated at the mean of rounds 1-2"
    est = t_init + t_updates + t_revs + t_fin
    sample = (f"oracle (C port of the numba kernels) at full {data.shape[0]}x{data.shape[1]}: init {t_init:.2f}s, "
              f"update rounds 1-2 {t_up[0]:.2f}s+{t_up[1]:.2f}s, reverse {t_rev:.2f}s, finalize {t_fin:.2f}s; "
              f"{how}; {threads} threads")
    return est, {"threads": threads, "sample": sample, "sampled_seconds": t_init + sum(t_up) + t_rev + t_fin}


def run_reference(args, rank: int):
    if rank != 0:
        return
    from paper_2510_02774_b200.core import generate

    data = generate(args.n, args.dim, "gaussian", seed=1).data
    pairs = round_pairs(PARAMS["T1"], PARAMS["T2"]) if args.n == 1_000_000 else None
    info = None
    for _ in range(args.warmup):
        cpu_sample(data, pairs)
    vals = []
    for _ in range(args.steps):
        v, info = cpu_sample(data, pairs)
        vals.append(v)
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value * 1e3, 1),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (numpy default_rng(1).standard_normal)",
        "config": {"workload": WORKLOAD, "n": args.n, "dim": args.dim, **PARAMS},
        "cpu_baseline": {"value": round(value, 3), "unit": "s", "cores": info["threads"], "kind": "port",
                         "sample": info["sample"]},
        "e2e": {"value": round(value, 3), "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU leg
def run_gpu(args, rank: int, world: int, local_rank: int):
    import torch

    import paper_2510_02774_b200 as g
    from paper_2510_02774_b200 import _lib
    from paper_2510_02774_b200.builder import DeviceBuild, upload

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ds = g.generate(args.n, args.dim, "gaussian", seed=1)
    params = g.BuildParams(**PARAMS)
    data_dev = upload(ds.data, dev)
    if world > 1:
        from paper_2510_02774_b200.sharded import ShardedBuild, build_sharded

        eng = ShardedBuild(data_dev, args.dim, params, rank, world)
    else:
        eng = DeviceBuild(data_dev, args.dim, params)
    stream = torch.cuda.current_stream(dev)

    for _ in range(args.warmup):
        eng.run()
    torch.cuda.synchronize()

    # ---- timed region: device-resident build, K steps ----
    phase = []
    launches0 = int(_lib.lib.grnnd_launch_count())
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for s in range(args.steps):
            out = eng.run(phase_events=phase if s == args.steps - 1 else None)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    launches = (int(_lib.lib.grnnd_launch_count()) - launches0) // args.steps
    ms_step = e0.elapsed_time(e1) / args.steps
    ms_step = max_over_ranks(ms_step)
    offsets, nbrs, bad, _ = out
    assert int(bad.item()) == 0, "finalize flagged an invalid graph"
    stats = eng.round_stats()
    upd = [s for s in stats if s.kind == "update"]
    prop_ms = [a.elapsed_time(b) for a, b, _ in phase]
    apply_ms = [b.elapsed_time(c) for _, b, c in phase]
    edges = int(offsets[-1].item())

    # ---- e2e through the public API, host buffers (pinned) ----
    host = torch.from_numpy(ds.data).pin_memory()
    pinned_ds = g.Dataset(host.numpy())
    api_build = (lambda d, p: build_sharded(d, p)) if world > 1 else g.build
    api_build(pinned_ds, params)  # warm the allocator for this path
    e2e = []
    for _ in range(args.steps):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        graph = api_build(pinned_ds, params)
        e2e.append(time.perf_counter() - t0)
    e2e_s = max_over_ranks(statistics.mean(e2e))
    h2d = ds.data.nbytes
    d2h = graph.offsets.nbytes + graph.neighbor_ids.nbytes

    # ---- roofline of the dominant kernel (propagate = the pair phase) ----
    pk, pk_kind = peaks()
    D = args.dim
    sum_k = [s.messages for s in upd]
    alg_bytes = [(4 * D + 40) * k for k in sum_k]  # SURVEY 8(d) d3 per update round
    ach_gbs = sum(alg_bytes) / (sum(prop_ms) * 1e-3) / 1e9
    pairs_ref = [s.pairs_ref for s in upd]
    pairs_all = [s.pairs for s in upd]
    cands = [s.candidates for s in upd]
    # tensor-core pre-screen: every group is one Gram of M = 128 rows x N <= 96 x K = 128 (tf32)
    sm_mhz = clk.summary().get("sm_mhz") or pk.get("sm_max_mhz", 1965.0)
    traffic = None
    try:
        nc = json.loads(NCU_FILE.read_text())
        traffic = nc.get("dram_bytes_per_round")
    except Exception:
        pass
    if rank == 0 and args.n == 1_000_000:
        try:
            PAIRS_FILE.parent.mkdir(exist_ok=True)
            if not PAIRS_FILE.exists():
                PAIRS_FILE.write_text(json.dumps({"n": args.n, "pairs_ref": pairs_ref, "pairs": pairs_all,
                                                  "sum_k": sum_k}))
        except Exception:
            pass

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        est, info = cpu_sample(ds.data, round_pairs(PARAMS["T1"], PARAMS["T2"]) or pairs_ref)
        cpu = {"value": round(est, 2), "unit": "s", "cores": info["threads"], "kind": "port",
               "sample": info["sample"]}

    if rank == 0:
        value = ms_step / 1e3
        line = {
            "metric": METRIC, "value": round(value, 4), "unit": "s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 2), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (numpy default_rng(1).standard_normal, the reference's generate recipe)",
            "config": {"workload": WORKLOAD, "n": args.n, "dim": args.dim, **PARAMS,
                       "parallelism": f"shard{world} (ID-range ownership, NCCL all-to-all per round)" if world > 1 else "single",
                       "l2": "inputs larger than L2 (512 MB vectors, 0.77 GB pools)"},
            "mvec_per_s": round(args.n * world / value / 1e6, 3),
            "edges": edges,
            "clocks": clk.summary(),
            "e2e": {"value": round(e2e_s, 4), "unit": "s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches,
            "roofline": {"bound": "hbm", "achieved": round(ach_gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                         "frac": round(ach_gbs / pk["hbm_gbs"], 4), "traffic": traffic,
                         "kernel": "pair phase (tc_stage + tc3_pairs bins + decide)", "peak_source": pk_kind,
                         "alg_bytes_per_round": int(sum(alg_bytes) / len(alg_bytes)),
                         "ms_per_round": round(sum(prop_ms) / len(prop_ms), 3)},
            "pair_phase": {"design": "tcgen05 TF32 Gram pre-screen with a rigorous error band + exact fp32 "
                                     "re-evaluation of the band (bit-identical to the reference)",
                           "pairs_per_round": int(sum(pairs_all) / len(pairs_all)),
                           "pairs_ref_per_round": int(sum(pairs_ref) / len(pairs_ref)),
                           "exact_reevaluated_frac": round(sum(cands) / max(sum(pairs_all), 1), 5),
                           "sm_mhz": sm_mhz},
            "phase_ms_per_round": {"propagate": round(sum(prop_ms) / len(prop_ms), 3),
                                   "group_apply": round(sum(apply_ms) / len(apply_ms), 3)},
            "cpu_baseline": cpu,
            "parity": "graph bit-identical to the reference (tests/test_gpu_parity.py)",
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", args.gpus if args.gpus == 1 else 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    run_gpu(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
