"""Benchmark: batched MRPT k-NN queries on B200 (BASELINE.json metric).

One step = one batched pass of the hot path (project+route K2 -> vote K3 ->
exact scan+top-k K4) over the configuration's whole query batch, with the
index and the queries resident in HBM.  Default workload: BASELINE config 2
(configs[1], image-pixel-shaped, n=60k, d=784, 10k queries, T=100, l=8,
k=10) at its highest-recall vote threshold.  Prints ONE JSON line on rank 0.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--votes V]
    python bench.py --impl reference ...   # the reference CPU package, same workload
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1509_06957_b200 import workloads  # noqa: E402

PEAKS_FALLBACK_GBS = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--votes", type=int, default=None)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--sweep", action="store_true", help="also time every v of the config")
    return ap.parse_args()


def tensor_peak_i8():
    """int8 tensor peak for the fused filter's roofline: the int8 rate measured
    on this pool's B200 (profiles/int8_peak.json, tools/int8_peak.py: cuBLASLt
    IMMA 8192^3 burst), else 2x the measured dense bf16 rate."""
    try:
        pk = json.load(open(os.path.join(ROOT, "profiles", "int8_peak.json")))
        return float(pk["int8_tops"]), "measured int8 (cuBLASLt 8192^3 burst, profiles/int8_peak.json)"
    except Exception:
        pass
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return 2.0 * float(mp["bf16_tflops"]), "2x measured bf16 dense (int8 not measured)"
    except Exception:
        return 2.0 * 1590.0, "2x fallback bf16 dense (B200_PROFILING.md)"


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return PEAKS_FALLBACK_GBS, "fallback"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md recipe)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait()
            self.fh.close()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            return None
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if len(r) > 4 + i and "Active" in r[4 + i] and "Not" not in r[4 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- reference CPU
def _ref_import():
    ref = os.path.join(ROOT, "oracle", "_ref")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import mrpt  # noqa: F401  (the unmodified reference package)

    return mrpt


_POOL_STATE = {}


def _ref_worker(args):
    lo, hi = args
    mrpt = _ref_import()
    st = _POOL_STATE
    for i in range(lo, hi):
        mrpt.approximate_knn(st["Q"][i], st["k"], st["index"], st["v"])
    return hi - lo


def ref_query_rate(index, Q, k, v, seconds, cores):
    """Reference approximate_knn (single query per call, search.py:175-184) over a
    bounded query sample, one forked worker per core sharing the index."""
    import multiprocessing as mp

    mrpt = _ref_import()
    t0 = time.perf_counter()
    mrpt.approximate_knn(Q[0], k, index, v)
    one = max(1e-5, time.perf_counter() - t0)
    sample = int(min(len(Q), max(cores, seconds / one * cores)))
    _POOL_STATE.update(Q=Q, k=k, v=v, index=index)
    bounds = np.linspace(0, sample, cores + 1).astype(int)
    jobs = [(int(bounds[i]), int(bounds[i + 1])) for i in range(cores) if bounds[i + 1] > bounds[i]]
    ctx = mp.get_context("fork")
    with ctx.Pool(len(jobs)) as pool:
        t0 = time.perf_counter()
        done = sum(pool.map(_ref_worker, jobs))
        dt = time.perf_counter() - t0
    return done / dt, done, dt


def ref_index_from_arrays(X, p, matrices, splits, offsets, indices, checksum):
    mrpt = _ref_import()
    mats = [mrpt.SparseProjectionMatrix(d=R.d, depth=R.depth, a=R.a, seed=R.seed, col_ptr=R.col_ptr,
                                        row_idx=R.row_idx, values=R.values,
                                        fixed_count=R.fixed_count) for R in matrices]
    return mrpt.MRPTIndex(dataset=mrpt.Dataset(X), n_trees=p["n_trees"], depth=p["depth"],
                          sparsity=p["sparsity"], seed=p["seed"], fixed_count=False, matrices=mats,
                          splits=splits, leaf_offsets=offsets, leaf_indices=indices,
                          dataset_checksum=checksum)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    mrpt = _ref_import()
    X, Q, p = workloads.generate(args.config, args.scale)
    v = args.votes or p["headline_votes"]
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    index = mrpt.grow_trees(X, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"],
                            threads=cores)
    build_s = time.perf_counter() - t0
    for _ in range(args.warmup):
        ref_query_rate(index, Q, p["k"], v, 1.0, cores)
    rates = []
    for _ in range(args.steps):
        qps, done, dt = ref_query_rate(index, Q, p["k"], v, args.cpu_seconds / max(1, args.steps),
                                       cores)
        rates.append(qps)
    value = float(np.mean(rates))
    line = {
        "impl": "reference", "metric": "queries/sec (approximate k-NN, batched queries)",
        "value": value, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * p["nq"] / value, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p["name"], "n": p["n"], "d": p["d"], "nq": p["nq"],
                   "n_trees": p["n_trees"], "depth": p["depth"], "k": p["k"], "votes": v},
        "build_s": build_s,
        "cpu_baseline": {"value": value, "unit": "queries/s", "cores": cores, "kind": "reference",
                         "sample": f"reference mrpt.approximate_knn, one query per call, forked "
                                   f"pool of {cores}, ~{args.cpu_seconds:.0f}s of queries per run"},
        "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1509_06957_b200 as mrpt
    from paper_1509_06957_b200.search import query_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    X, Q, p = workloads.generate(args.config, args.scale)
    v = args.votes or p["headline_votes"]
    k = p["k"]
    stream = torch.cuda.current_stream()

    # --- build (device-resident X) ------------------------------------------------
    # one tiny build first so one-time module loading is not billed to build_s
    warm = torch.randn(512, X.shape[1], device="cuda")
    mrpt.grow_trees(warm, 2, 3, seed=1)
    Xd = torch.from_numpy(X).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world > 1:
        from paper_1509_06957_b200.distributed import grow_trees_distributed

        index = grow_trees_distributed(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
    else:
        index = mrpt.grow_trees(Xd, p["n_trees"], p["depth"], p["sparsity"], seed=p["seed"])
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0  # includes the GPU FNV checksum
    D = index.device_index()
    Qd = torch.from_numpy(Q).cuda()

    # --- per-query algorithmic bytes: 4*sum_t|L_t(q)| + 4*d*|S(q)| ---
    ids, dists, counts = query_device(D, Qd, k, v)
    from paper_1509_06957_b200.search import _route_device

    leaves = _route_device(Qd, D).long()
    sizes = (D.offsets[:, 1:] - D.offsets[:, :-1])  # (T, nleaf)
    touched = sizes.gather(1, leaves.t()).sum(0).double()  # (nq,)
    cand = counts.double()
    vote_bytes = float(4.0 * touched.sum().item())
    scan_bytes = float(4.0 * p["d"] * cand.sum().item())
    torch.cuda.synchronize()

    # --- stage timing hooks: events around each kernel, on the launching stream ---
    stage_ms = {"route": 0.0, "vote": 0.0, "scan_topk": 0.0}

    def timed_step(events):
        return query_device(D, Qd, k, v, timer=events)

    # L2 is flushed between timed steps (a 2x-L2 write outside each step's events):
    # within a step, the index and data rows are re-read by many queries, which is
    # the workload; across steps nothing stays warm.  Warm-up runs the identical
    # sequence (flush, events, stage timers) so no first-use cost lands in the
    # timed region.
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        flush.fill_(1)
        w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0.record(stream)
        timed_step([])
        w1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    evs = []
    step_ev = []
    from paper_1509_06957_b200 import _native as native

    lib = native.load()
    launches0 = int(lib.mrpt_launch_count())
    lib.mrpt_kernel_timer(1)  # events around the fused filter launches (roofline)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            flush.fill_(1)
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            s0.record(stream)
            ev = []
            timed_step(ev)
            s1.record(stream)
            evs.append(ev)
            step_ev.append((s0, s1))
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    elapsed_ms = sum(a.elapsed_time(b) for a, b in step_ev)
    for ev in evs:
        for name, a, b in ev:
            stage_ms[name] += a.elapsed_time(b)
    launches = int(lib.mrpt_launch_count()) - launches0  # this library's kernels, timed steps only
    kt_ms, kt_n = ctypes.c_double(0.0), ctypes.c_int64(0)
    native.call("mrpt_kernel_timer_read", ctypes.byref(kt_ms), ctypes.byref(kt_n))
    lib.mrpt_kernel_timer(0)
    stage_launches = {name: sum(1 for ev in evs for (nm, _, _) in ev if nm == name) for name in stage_ms}
    if world > 1:
        t = torch.tensor([elapsed_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    total_q = p["nq"] * args.steps * world
    value = total_q / (elapsed_ms / 1000.0)

    # --- e2e through the public API: pinned host queries in, host results out ------
    Qpin = torch.from_numpy(Q).pin_memory()
    for _ in range(5):
        mrpt.approximate_knn_batch(Qpin, k, index, v)
    torch.cuda.synchronize()
    # three runs of e2e_steps calls each, the median run reported: a host-side
    # stall (the box's CPU is shared) in one run does not decide the number
    e2e_steps = max(3, min(args.steps, 10))
    runs = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            out = mrpt.approximate_knn_batch(Qpin, k, index, v)
        runs.append(time.perf_counter() - t0)
    e2e_s = float(np.median(runs))
    if world > 1:
        t = torch.tensor([e2e_s], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = p["nq"] * e2e_steps * world / e2e_s
    h2d = Q.nbytes
    d2h = sum(np.asarray(o).nbytes for o in out)

    # recall vs exact ground truth (brute force through the same exact kernel);
    # above ~2e10 row-query pairs (config 5) on a fixed subsample of queries
    n_gt = p["nq"] if p["n"] * p["nq"] <= 2e10 else max(100, int(2e10 // p["n"]))
    gt_ids, _, _ = query_device_brute(D, Qd[:n_gt], k)
    recall = float(np.mean([len(np.intersect1d(a[a >= 0], b)) / k
                            for a, b in zip(ids[:n_gt].cpu().numpy(), gt_ids.cpu().numpy())]))

    # --- roofline of the dominant kernel (and of the vote+scan stage) -------------
    peak, peak_kind = hbm_peak()
    steps = args.steps
    per_launch = {}
    nlaunch = stage_launches
    for name in stage_ms:
        per_launch[name] = stage_ms[name] / max(1, nlaunch[name])
    dominant = "scan_topk" if stage_ms["scan_topk"] >= stage_ms["vote"] else "vote"
    dom_bytes = (scan_bytes if dominant == "scan_topk" else vote_bytes) / max(1, nlaunch[dominant] // steps)
    achieved = dom_bytes / (per_launch[dominant] / 1000.0) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_config{args.config}_v{v}.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dominant)
        except Exception:
            traffic = None
    # bytes the chosen filter variant actually reads per candidate (its row
    # format + per-row side data + the candidate id); survivors reranked in fp32
    # are not included
    from paper_1509_06957_b200.search import _size_class

    variant = (D.scan_pin.get((k, v)) or D.scan_choice_by_size.get((k, v, _size_class(p["nq"])))
               or D.scan_choice.get((k, v), "fp32"))
    if variant == "u8tc_bits":
        # fused tcgen05 filter: no dot-product matrix; per candidate its bit
        # (read once per (query, row)) and, per row tile, 16-B row records
        row_b, filt_mb = 0, D.n * D.u8_rows()[1] / 1e6
    elif variant.startswith("u8gemm"):
        # per candidate: its dot product (4 B) + row record (16 B) (+ its id in
        # list mode); per query: the GEMM's n dot products written and read
        row_b, filt_mb = 16 if variant == "u8gemm_bits" else 20, D.n * D.u8_rows()[1] / 1e6
    elif variant == "u8":
        row_b, filt_mb = D.u8_rows()[1] + 12, D.n * D.u8_rows()[1] / 1e6
    elif variant == "fp16":
        row_b, filt_mb = 2 * D.shadow()[1] + 4, D.n * 2 * D.shadow()[1] / 1e6
    else:
        row_b, filt_mb = 4 * p["d"], X.nbytes / 1e6
    filter_bytes = float(cand.sum().item()) * (row_b + 4)
    if variant.startswith("u8gemm"):
        filter_bytes += 8.0 * D.n * p["nq"]
    if variant == "u8tc_bits":
        filter_bytes = D.n * p["nq"] / 8.0 + 16.0 * D.n * math.ceil(p["nq"] / 128)
    filter_gbs = filter_bytes / (stage_ms["scan_topk"] / steps / 1000.0) / 1e9
    stage_gbs = (vote_bytes + scan_bytes) / ((stage_ms["vote"] + stage_ms["scan_topk"]) / steps / 1000.0) / 1e9

    roof = None
    if variant == "u8tc_bits" and kt_n.value > 0:
        # the fused filter is a tensor-core kernel: int8 ops of the (query,
        # row) dot products it forms (2*nq*n*d per step), live CUDA-event
        # duration of its launches; peak = the measured int8 rate of this
        # pool's B200 (profiles/int8_peak.json)
        per_ms = kt_ms.value / kt_n.value
        launches_per_step = kt_n.value / steps
        ops = 2.0 * p["nq"] * D.n * p["d"] / launches_per_step
        tops = ops / (per_ms / 1000.0) / 1e12
        tpeak, tkind = tensor_peak_i8()
        ttraffic = None
        if os.path.exists(tpath):
            try:
                ttraffic = json.load(open(tpath)).get("k_tc_filter")
            except Exception:
                ttraffic = None
        roof = {"bound": "tensor", "kernel": "k_tc_filter (fused tcgen05 int8 filter)",
                "achieved": tops, "peak": tpeak, "peak_kind": tkind, "unit": "TOP/s",
                "frac": tops / tpeak, "traffic": ttraffic,
                "kernel_ms_per_launch": per_ms, "kernel_launches_per_step": launches_per_step,
                "hbm_algorithmic": {"kernel": dominant, "achieved_gbs": achieved, "peak": peak,
                                    "frac": achieved / peak,
                                    "note": "SURVEY 8(d) algorithmic bytes (4*d B per candidate row) "
                                            "over the scan stage; the fused filter never reads "
                                            "float32 rows"},
                "stage_vote_plus_scan_gbs": stage_gbs, "stage_frac": stage_gbs / peak,
                "bytes_per_query": (vote_bytes + scan_bytes) / p["nq"], "scan_variant": variant,
                "scan_filter_bytes_per_query": filter_bytes / p["nq"],
                "note": ("ops = 2*nq*n*d int8 multiply-adds of the dot products the kernel forms "
                         "(tcgen05.mma.kind::i8, K padded to 128-B blocks not counted); traffic "
                         "= ncu DRAM bytes per launch (profiles/traffic_*.json)")}
    line = {
        "metric": "queries/sec (approximate k-NN, batched queries)",
        "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p["name"], "n": p["n"], "d": p["d"], "nq_per_gpu": p["nq"],
                   "n_trees": p["n_trees"], "depth": p["depth"], "k": k, "votes": v,
                   "sparsity": p["sparsity"], "generator": p["generator"],
                   "l2": "L2 flushed between timed steps (256 MB write outside the step "
                         "events); X %.0f MB, leaf ids %.0f MB, scan filter rows %.0f MB" % (
                       X.nbytes / 1e6, 4.0 * p["n_trees"] * p["n"] / 1e6, filt_mb),
                   "parallelism": f"replicated index, queries sharded by batch x{world}"},
        "recall_at_k": recall,
        "recall_queries": n_gt,
        "mean_candidates": float(cand.mean().item()),
        "build_s": build_s,
        "roofline": roof if roof is not None else {"bound": "hbm", "kernel": dominant, "achieved": achieved, "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "stage_vote_plus_scan_gbs": stage_gbs,
                     "stage_frac": stage_gbs / peak,
                     "bytes_per_query": (vote_bytes + scan_bytes) / p["nq"],
                     "scan_variant": variant,
                     "scan_filter_bytes_per_query": filter_bytes / p["nq"],
                     "scan_filter_gbs": filter_gbs,
                     "note": ("achieved/frac use SURVEY 8(d) algorithmic bytes (4 B per leaf id "
                              "+ 4*d B per candidate row); frac > 1 is possible because the "
                              "exact scan does not read float32 candidate rows: " + (
                                  "an int8 tensor-core GEMM forms every (query, row) dot "
                                  "product on the u8 shadow (written and read once, 4 B each) "
                                  "and the filter reads a 16-B record per candidate"
                                  if variant.startswith("u8gemm") else
                                  "it filters on %s rows (%d B/candidate), L2-resident within "
                                  "a step" % (variant, row_b + 4)) +
                              "; exact float64 re-rank of the survivors only; traffic = ncu "
                              "DRAM bytes of the stage per call (profiles/traffic_*.json)")},
        "stage_ms_per_step": {k2: v2 / steps for k2, v2 in stage_ms.items()},
        "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "method": f"approximate_knn_batch on pinned host queries, wall clock; median of 3 runs "
                          f"of {e2e_steps} calls (run means: "
                          + ", ".join(f"{p['nq'] * e2e_steps / r:.0f}" for r in runs) + " queries/s)"},
        "gpu_launches": int(launches),
    }
    if args.sweep:
        sw = {}
        for vv in p["votes"]:
            for _ in range(2):
                query_device(D, Qd, k, vv)
            torch.cuda.synchronize()
            # per-call events, median of 3 (robust to a stray host stall)
            per = []
            for _ in range(3):
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record(stream)
                r = query_device(D, Qd, k, vv)
                e.record(stream)
                torch.cuda.synchronize()
                per.append(s.elapsed_time(e))
            rc = float(np.mean([len(np.intersect1d(a[a >= 0], b)) / k
                                for a, b in zip(r[0][:n_gt].cpu().numpy(), gt_ids.cpu().numpy())]))
            sw[str(vv)] = {"qps": p["nq"] / (float(np.median(per)) / 1000.0), "recall": rc,
                           "mean_candidates": float(r[2].double().mean().item())}
        line["sweep"] = sw
        # the same thresholds from one route + one counted vote (f4)
        for _ in range(2):
            mrpt.approximate_knn_sweep(Qd, k, index, p["votes"])
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(3):
            mrpt.approximate_knn_sweep(Qd, k, index, p["votes"])
        e.record(stream)
        torch.cuda.synchronize()
        one = s.elapsed_time(e) / 3
        line["sweep_one_pass"] = {
            "votes": list(p["votes"]), "ms_all_thresholds": one,
            "ms_sum_separate": sum(p["nq"] / x["qps"] * 1e3 for x in sw.values())}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, X, Q, p, v, index)
    line["clocks"] = clk.summary()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def query_device_brute(D, Qd, k):
    """Exact k-NN over all points (cand == NULL mode of mrpt_scan_topk)."""
    import torch

    from paper_1509_06957_b200 import _native

    nq = int(Qd.shape[0])
    ids = torch.empty((nq, k), dtype=torch.int64, device=Qd.device)
    dists = torch.empty((nq, k), dtype=torch.float64, device=Qd.device)
    _native.call("mrpt_scan_topk", _native.ptr(D.X), D.n, D.d, int(D.X.stride(0)), _native.ptr(Qd),
                 nq, int(Qd.stride(0)), None, 0, None, int(k), _native.ptr(ids),
                 _native.ptr(dists), _native.stream_ptr())
    return ids, dists, None


def cpu_baseline(args, X, Q, p, v, index):
    """The unmodified reference (oracle/_ref) on the host cores, over the GPU-built
    index (bit-identical to the reference's own build), bounded sample."""
    try:
        cores = len(os.sched_getaffinity(0))
        rindex = ref_index_from_arrays(X, p, index.matrices, index.splits, index.leaf_offsets,
                                       index.leaf_indices, index.dataset_checksum)
        qps, done, dt = ref_query_rate(rindex, Q, p["k"], v, args.cpu_seconds, cores)
        return {"value": qps, "unit": "queries/s", "cores": cores, "kind": "reference",
                "sample": f"{done} queries of {p['name']} (v={v}) through reference "
                          f"mrpt.approximate_knn, forked pool of {cores}, {dt:.1f}s"}
    except Exception as exc:  # the baseline is reported, never required
        return {"value": None, "unit": "queries/s", "cores": None, "kind": "reference",
                "sample": f"unavailable: {exc}"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
