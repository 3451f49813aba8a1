"""Benchmark of the MinHash-LSH hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (BASELINE.json configs[1], "C2"): per GPU 1,000,000 synthetic
documents of 1600-2400 bytes (mean ~2 KB, 37-char alphabet, 5% of docs in
near-duplicate pairs at edit rate 1/100), 5-byte shingles, H=128 hashes,
16 bands x 8 rows, K=2000.  A step = signatures + band keys for the whole
shard.  Shards are independent (weak scaling, no data-path collective).

Printed JSON (one line, rank 0):
  value     docs/s, inputs resident in HBM (device entry point, CUDA events on
            the launching stream, max over ranks)
  e2e       same metric through the public host entry point nd_signatures with
            pinned host buffers: H2D of text+offsets and D2H of signatures+band
            keys inside every timed step
  dedup     end-to-end in-memory dedup docs/s (host buffers -> report) on the
            same shard (secondary metric of BASELINE.json)
  roofline  K1 (signature kernel) vs the integer-issue roofline
            (8 int ops per hash-window evaluation) and vs HBM
  staged    the reference's file-backed workflow end to end on the first
            200k documents written as JSONL: C++ loader (parse + NFC + filters),
            K1 -> .feds, .feds -> HBM -> K2/K3 -> .pairs, K4 -> report, i.e.
            run_dedup's three stages with every artifact on disk (wall clock,
            rank 0 at N=1), plus the loader's own docs/s
  cpu_baseline  the reference implementation (oracle/_ref: the reference's own
            sources compiled in place) on this host's cores, bounded sample
--impl reference times only the reference CPU path (oracle/_ref) on the same
workload/metric and prints the same line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import ctypes as C
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

DOCS = 1_000_000
H, BANDS, ROWS, L = 128, 16, 8, 5
LEN_MIN, LEN_MAX = 1600, 2400
OPS_PER_HWE = 8  # the paper's Eq.5 update made exact on 32-bit integer instructions
METRIC = "MinHash signatures docs/sec and end-to-end dedup docs/sec at 1/2/4/8 B200"
WORKLOAD = ("C2: 1M synthetic docs/GPU, 1600-2400 B (37-char alphabet), 10% near-dups "
            "(pairs, edit 1/100), 5-byte shingles, 128 hashes, 16x8 bands, K=2000; "
            "signature gen + banding")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--docs", type=int, default=DOCS)
    ap.add_argument("--no-dedup", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-staged", action="store_true")
    ap.add_argument("--staged-docs", type=int, default=200_000)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def make_corpus(lib, docs: int, seed: int, pinned: bool):
    """Deterministic C2-shaped shard (nd_synth_generate mode 1, multi-threaded)."""
    from paper_2501_01046_b200 import _lib

    spec = _lib.NdSynthSpec(doc_count=docs, group_count=docs // 20, group_size_min=2,
                            group_size_max=2, edit_num=1, edit_den=100, len_min=LEN_MIN,
                            len_max=LEN_MAX, seed=seed, mode=1)
    nb = C.c_uint64()
    _lib.check(lib.nd_synth_generate(C.byref(spec), None, None, C.byref(nb)))
    if pinned:
        import torch

        data = torch.empty(nb.value, dtype=torch.uint8, pin_memory=True).numpy()
        offs = torch.empty(docs + 1, dtype=torch.int64, pin_memory=True).numpy().view(np.uint64)
    else:
        data = np.empty(nb.value, np.uint8)
        offs = np.empty(docs + 1, np.uint64)
    _lib.check(lib.nd_synth_generate(C.byref(spec), data.ctypes.data_as(_lib.u8p),
                                     offs.ctypes.data_as(_lib.u64p), C.byref(nb)))
    return data, offs


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 4 + i and s[4 + i].lower().startswith("active")})
        loaded = [x for x in sm if x > 0.5 * (max(mx) if mx else 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def cpu_reference_rate(data, offs, sample_docs: int, workers: int):
    """Reference signature_of_document + band_bucket_ids (oracle/_ref) on host cores."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Ref  # the reference itself, compiled in place

    ref = Ref()
    n = min(sample_docs, len(offs) - 1)
    sub_offs = offs[: n + 1].copy()
    sub = data[: int(sub_offs[-1])]
    t = time.perf_counter()
    ref.signatures(sub, sub_offs, seed=5, H=H, L=L, bands=BANDS, rows=ROWS, K=2000,
                   workers=workers)
    dt = time.perf_counter() - t
    return n / dt, n, dt


def cpu_reference_dedup_rate(data, offs, docs: int, workers: int):
    """The reference's own run_dedup (all three stages, oracle/_ref) on the
    first `docs` documents written as JSONL, on the host cores: the CPU
    counterpart of the `dedup` and `staged` lines."""
    import shutil
    import tempfile

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_bind import Ref

    ref = Ref()
    tmp = tempfile.mkdtemp(prefix="nd_refdedup_")
    try:
        src = os.path.join(tmp, "c.jsonl")
        raw = np.asarray(data[:int(offs[docs])]).tobytes()
        o = offs[:docs + 1].astype(np.int64)
        with open(src, "wb") as f:
            f.write(b"".join(b'{"text":"' + raw[o[i]:o[i + 1]] + b'"}\n' for i in range(docs)))
        ws = os.path.join(tmp, "ws")
        os.makedirs(ws)
        t = time.perf_counter()
        ref.run_dedup(src, ws, workers=workers, memory_budget=64 << 30)
        dt = time.perf_counter() - t
        return docs / dt, dt
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def calibrate_cpu_sample(data, offs, workers: int, target_s: float):
    rate, _, _ = cpu_reference_rate(data, offs, max(256, 64 * workers), workers)
    return int(min(len(offs) - 1, max(512, rate * target_s)))


def run_reference(args, world, rank):
    """--impl reference: the reference's CPU path on this host's cores."""
    if rank != 0:
        return
    from paper_2501_01046_b200 import _lib

    lib = _lib.load()
    data, offs = make_corpus(lib, min(args.docs, 200_000), 1, pinned=False)
    workers = os.cpu_count() or 1
    sample = calibrate_cpu_sample(data, offs, workers, 3.0)
    for _ in range(args.warmup):
        cpu_reference_rate(data, offs, min(sample, 512), workers)
    total_docs, total_t = 0, 0.0
    for _ in range(args.steps):
        _, n, dt = cpu_reference_rate(data, offs, sample, workers)
        total_docs += n
        total_t += dt
    value = total_docs / total_t
    line = {"metric": METRIC, "impl": "reference", "value": value, "unit": "docs/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * total_t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "docs_per_step": sample},
            "cpu_baseline": {"value": value, "unit": "docs/s", "cores": workers,
                             "kind": "reference",
                             "sample": f"{sample} docs of the C2 shard per step "
                                       "(signature_of_document + band_bucket_ids via "
                                       "parallel_for_index, oracle/_ref)"},
            "e2e": {"value": value, "unit": "docs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_staged(data, offs, docs: int):
    """JSONL -> workspace through the staged workflow (pipeline.run_dedup)."""
    import shutil
    import tempfile

    from paper_2501_01046_b200 import corpus, pipeline

    docs = min(docs, len(offs) - 1)
    tmp = tempfile.mkdtemp(prefix="nd_staged_")
    try:
        src = os.path.join(tmp, "corpus.jsonl")
        raw = np.asarray(data[:int(offs[docs])]).tobytes()
        with open(src, "wb") as f:
            o = offs[:docs + 1].astype(np.int64)
            f.write(b"".join(b'{"text":"' + raw[o[i]:o[i + 1]] + b'"}\n' for i in range(docs)))
        jsonl_bytes = os.path.getsize(src)
        cfg = pipeline.RunConfig(inputs=[src], workspace=os.path.join(tmp, "ws"))
        t0 = time.perf_counter()
        f = corpus.JsonlFile(src, cfg, keep_text=True)
        f.packed(0)
        t_load = time.perf_counter() - t0
        f.close()
        pipeline.run_dedup(cfg)  # warm-up (allocations, page cache)
        shutil.rmtree(cfg.workspace)
        t = {}
        t0 = time.perf_counter()
        rep = pipeline.run_dedup(cfg, timings=t)
        wall = time.perf_counter() - t0
        return {"value": docs / wall, "unit": "docs/s", "docs": docs, "jsonl_bytes": jsonl_bytes,
                "seconds": wall, "hash_seconds": t["hash_seconds"],
                "compare_seconds": t["compare_seconds"], "union_seconds": t["union_seconds"],
                "groups": len(rep.groups), "distinct_pairs": rep.distinct_pairs,
                "loader": {"value": docs / t_load, "unit": "docs/s",
                           "gb_per_s": jsonl_bytes / t_load / 1e9, "threads": os.cpu_count()},
                "note": "pipeline.run_dedup: C++ JSONL loader, K1 -> .feds, compare stage -> "
                        ".pairs, union stage -> report; wall clock incl. file I/O"}
    finally:
        shutil.rmtree(tmp, ignore_errors=True)


def load_traffic():
    """dram bytes per K1 launch from the committed ncu --set full capture."""
    p = os.path.join(ROOT, "profiles", "k1_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def main():
    args = parse()
    world, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, world, rank)
        return
    import torch

    # one rank per GPU over NCCL; ND_DIST_BACKEND=gloo lets several ranks
    # share one GPU (harness check of the multi-rank path, not a measurement)
    backend = os.environ.get("ND_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend == "gloo" else local
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2501_01046_b200 import _lib, minhash
    from paper_2501_01046_b200.device import Context

    lib = _lib.load()
    docs = args.docs
    data, offs = make_corpus(lib, docs, 1 + 7919 * rank, pinned=True)
    nbytes = int(offs[-1])
    lens = np.diff(offs).astype(np.float64)
    hwe = float(((lens - L + 1) * H).sum())
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = Context(local, stream=stream.cuda_stream)
    fam = minhash.derive_family(5, H, L)
    K = 2000

    # ---- value: device-resident inputs --------------------------------------
    d_data = torch.from_numpy(data).to("cuda", non_blocking=False)
    d_offs = torch.from_numpy(offs.view(np.int64)).to("cuda")
    d_sig = torch.empty((docs, H), dtype=torch.int32, device="cuda")
    d_band = torch.empty((docs, BANDS), dtype=torch.int32, device="cuda")

    def step_device():
        minhash.signatures_device(d_data.data_ptr(), d_offs.data_ptr(), docs, fam,
                                  d_sig.data_ptr(), d_band.data_ptr(), BANDS, ROWS, K, ctx=ctx)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step_device()
    barrier()
    launches0 = lib.nd_launch_count()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            step_device()
            ev[i][1].record(stream)
        t_end.record(stream)
        barrier()
    launches = lib.nd_launch_count() - launches0
    ms = max_over_ranks(t_start.elapsed_time(t_end))
    step_ms = [a.elapsed_time(b) for a, b in ev]
    value = world * docs * args.steps / (ms / 1e3)

    # ---- e2e: host pinned buffers through the public entry point -------------
    sig_h = torch.empty((docs, H), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    band_h = torch.empty((docs, BANDS), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)

    def step_host():
        minhash.signatures_packed(data, offs, fam, BANDS, ROWS, K, ctx=ctx, sig_out=sig_h,
                                  band_out=band_h)

    for _ in range(max(1, args.warmup)):
        step_host()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        step_host()
    e1.record(stream)
    barrier()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = world * docs * args.steps / (e2e_ms / 1e3)
    parity_host_device = bool(np.array_equal(sig_h, d_sig.cpu().numpy().view(np.uint32)))

    # ---- dedup: end-to-end in-memory dedup (host buffers -> report) ----------
    dedup = None
    if not args.no_dedup:
        try:
            from paper_2501_01046_b200 import pipeline

            if world > 1:
                from paper_2501_01046_b200 import distributed

                stages = distributed.GpuStages(ctx, torch.device("cuda", local))
                cfg = pipeline.RunConfig()
                distributed.dedup_sharded(data, offs, cfg, stages, fetch="arrays")  # warm-up
                barrier()
                reps = max(1, min(3, args.steps))
                d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                d0.record(stream)
                for _ in range(reps):
                    res = distributed.dedup_sharded(data, offs, cfg, stages, fetch="arrays")
                d1.record(stream)
                barrier()
                dms = max_over_ranks(d0.elapsed_time(d1) / reps)
                # one more run with the collectives timed on the device
                tm = {}
                distributed.dedup_sharded(data, offs, cfg, stages, fetch="arrays", timings=tm)
                xms = max_over_ranks(tm["exchange_ms"])
                ems = max_over_ranks(tm["edges_ms"])
                xbytes = max_over_ranks(float(tm["exchange_sent_bytes"]))
                dedup = {"value": world * docs / (dms / 1e3), "unit": "docs/s", "ms_per_run": dms,
                         "distinct_pairs": res.distinct_pairs, "candidate_pairs": res.candidate_pairs,
                         "emitted_pairs": res.emitted_pairs, "documents": res.documents,
                         "all_to_all": {"ms": xms, "max_bytes_sent_per_rank": xbytes,
                                        "bus_gb_s": xbytes / (xms / 1e3) / 1e9 if xms else None,
                                        "note": "cell-record exchange (keys + rows), device time "
                                                "max over ranks; bus GB/s = bytes a rank sends "
                                                "to its peers / time (NVLink 5: 900 GB/s per "
                                                "direction)"},
                         "edges_all_gather": {"ms": ems, "bytes": tm["edges_bytes"]},
                         "note": f"sharded dedup over {world} GPUs (NCCL all-to-all of cell "
                                 "records, all-gather of signatures and edges), pinned host "
                                 "shards -> groups on rank 0"}
            elif hasattr(pipeline, "dedup_packed"):
                cfg = pipeline.RunConfig()
                pipeline.dedup_packed(data, offs, cfg, ctx=ctx, fetch="arrays")  # warm-up
                barrier()
                reps = max(1, min(5, args.steps))
                d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                d0.record(stream)
                for _ in range(reps):
                    rep = pipeline.dedup_packed(data, offs, cfg, ctx=ctx, fetch="arrays")
                d1.record(stream)
                barrier()
                dms = d0.elapsed_time(d1) / reps
                st = rep.stats
                dedup = {"value": docs / (dms / 1e3), "unit": "docs/s", "ms_per_run": dms,
                         "groups": st["duplicate_groups"], "near_duplicates": st["near_duplicates"],
                         "distinct_pairs": st["distinct_pairs"],
                         "candidate_pairs": st["candidate_pairs"],
                         "emitted_pairs": st["emitted_pairs"], "cells": st["nonsingleton_cells"],
                         "stage_seconds": {"h2d+k1_signatures": st["seconds"][0],
                                           "k2_cells": st["seconds"][1],
                                           "k3_compare+k4_unique": st["seconds"][2],
                                           "k4_components": st["seconds"][4]},
                         "candidate_pairs_per_s": st["candidate_pairs"] / st["seconds"][2]
                         if st["seconds"][2] else None,
                         "note": "in-memory run_dedup equivalent per GPU shard: pinned host "
                                 "packed batch -> groups in host memory (H2D, K1-K4, D2H)"}
        except ImportError:
            dedup = None

    # ---- roofline of K1 --------------------------------------------------------
    clocks = clk.summary()
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        pass
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    f_run = (clocks.get("sm_mhz") or peaks.get("sm_max_mhz") or 1965.0) * 1e6
    f_max = (peaks.get("sm_max_mhz") or clocks.get("sm_max_mhz") or 1965.0) * 1e6
    k1_ms = statistics.mean(step_ms)  # one K1 launch (+ a tiny plan kernel) per step
    ops = OPS_PER_HWE * hwe
    achieved = ops / (k1_ms / 1e3) / 1e12
    peak_run = sms * 128 * f_run / 1e12
    peak_max = sms * 128 * f_max / 1e12
    hbm_bytes = nbytes + 8 * (docs + 1) + 4 * docs * (H + BANDS)
    hbm_gbs = hbm_bytes / (k1_ms / 1e3) / 1e9
    hbm_peak = peaks.get("hbm_gbs", 6544.3)
    traffic_info = load_traffic()
    traffic = traffic_info.get("bytes_per_launch") if traffic_info else None
    roofline = {"bound": "int_alu", "achieved": achieved, "peak": peak_run,
                "unit": "T int-ops/s", "frac": achieved / peak_run, "traffic": traffic,
                "traffic_unit": "dram bytes per launch (ncu --set full, profiles/k1_traffic.json)",
                "work": f"{OPS_PER_HWE} int ops x {hwe:.4g} hash-window evals per launch "
                        "(sum over docs of (len-L+1)*H)",
                "peak_basis": f"{sms} SMs x 128 lanes x measured SM clock "
                              f"{f_run / 1e6:.0f} MHz (integer issue; no int peak in "
                              "MEASURED_PEAKS.json)",
                "hwe_per_s": hwe / (k1_ms / 1e3),
                "frac_at_max_clock": achieved / peak_max,
                "hbm": {"achieved": hbm_gbs, "peak": hbm_peak, "unit": "GB/s",
                        "frac": hbm_gbs / hbm_peak, "bytes_per_launch": hbm_bytes,
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"}}

    staged = None
    if rank == 0 and world == 1 and not args.no_staged:
        try:
            staged = run_staged(data, offs, args.staged_docs)
        except Exception as e:  # reported, not required
            staged = {"value": None, "error": str(e)[:200]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            workers = os.cpu_count() or 1
            sample = calibrate_cpu_sample(data, offs, workers, 10.0)
            rate, n, dt = cpu_reference_rate(data, offs, sample, workers)
            cpu = {"value": rate, "unit": "docs/s", "cores": workers, "kind": "reference",
                   "sample": f"first {n} docs of the C2 shard ({dt:.1f} s): reference "
                             "signature_of_document + band_bucket_ids, parallel_for_index"}
        except Exception as e:  # the baseline is reported, not required
            cpu = {"value": None, "unit": "docs/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {e}"}
        if dedup is not None:
            try:
                n = min(50_000, docs)
                rate, dt = cpu_reference_dedup_rate(data, offs, n, os.cpu_count() or 1)
                dedup["cpu_baseline"] = {
                    "value": rate, "unit": "docs/s", "cores": os.cpu_count(), "kind": "reference",
                    "sample": f"reference run_dedup (JSONL -> report, all stages) on the first {n} "
                              f"docs of the shard ({dt:.1f} s)"}
            except Exception as e:
                dedup["cpu_baseline"] = {"value": None, "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "docs/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "u32", "data": "synthetic",
                "config": {"workload": WORKLOAD, "docs_per_gpu": docs, "hashes": H,
                           "bands": BANDS, "rows": ROWS, "shingle_len": L, "bucket_count": K,
                           "text_bytes_per_gpu": nbytes,
                           "l2": "inputs larger than L2 (text per step >> 126 MB)",
                           "parallelism": f"shard{world}"},
                "e2e": {"value": e2e_value, "unit": "docs/s",
                        "h2d_bytes_per_step": nbytes + 8 * (docs + 1),
                        "d2h_bytes_per_step": 4 * docs * (H + BANDS),
                        "parity_host_vs_device": parity_host_device},
                "dedup": dedup, "staged": staged, "roofline": roofline, "cpu_baseline": cpu,
                "clocks": clocks, "gpu_launches": int(launches),
                "kernel_ms": {"k1_mean": k1_ms, "k1_min": min(step_ms), "k1_max": max(step_ms)}}
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
