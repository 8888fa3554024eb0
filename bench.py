#!/usr/bin/env python
"""Benchmark of the learned-cache serve path (BASELINE.json metric: requests/s
and p50/p99 latency with learned caches vs no-cache; hit rate).

Default workload = the north star's target, BASELINE.json configs[2]:
ResNet-50 ImageNet 224x224 with a learned cache (Pool(C) = GAP head + FC(16)
selector) after each of the 16 bottleneck blocks, batch 128 per GPU, synthetic
weights and N(0,1) images, selectors calibrated to the paper's R50 exit profile
(1.53 % of requests run the full model). One step = one
batch through the serve path on every GPU. configs[1] (ResNet-18 CIFAR, batch
256) is `--config resnet18_cifar`.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config resnet18_cifar|c1_mlp|resnet50|vgg16_cifar|resnet152]
                  [--batch B] [--precision bf16x3|bf16]

N > 1: launched by torchrun, one process per GPU; each rank serves its own
request shard (pure request-level data parallelism, no collectives on the
hot path); the reported time is the max over ranks.
--impl reference: the reference's CPU path on this box's host cores
(oracle/_ref for the block-MLP config; the oracle port for CNN configs whose
base layers the reference does not implement), rank 0 only.
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

CONFIGS = {
    # name: (family, arch/spec, classes, default batch, full-DNN fraction, BASELINE config string)
    "resnet18_cifar": ("cnn", "resnet18_cifar", 10, 256, 0.0351,
                       "ResNet-18 CIFAR-10 with learned caches, batch 256, 1xB200"),
    "resnet50": ("cnn", "resnet50", 1000, 128, 0.0153,
                 "ResNet-50 ImageNet 224x224 with learned caches at 16 blocks, batch 128"),
    "resnet152": ("cnn", "resnet152", 1000, 512, 0.1532, "ResNet-152 ImageNet with learned caches, batch 512"),
    "vgg16_cifar": ("cnn", "vgg16_cifar", 10, 256, 0.05, "VGG-16 CIFAR-10 with FC+pool cache models"),
    "c1_mlp": ("mlp", None, 10, 256, 0.15,
               "ResNet-18 CIFAR-10 shape block-MLP (reference family), cache after every block"),
}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()
            while not self.rows and time.time() - t0 < 3.0:  # sampling is live before timing starts
                time.sleep(0.02)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def build_deployment(cfg_name, batch, precision, device, seed=2101):
    import paper_2101_07344_b200 as lcb
    from paper_2101_07344_b200.synthetic import (C1_MENU, C1_WIDTHS, calibrate_variants, image_inputs,
                                                 mlp_inputs)
    family, arch, classes, _, full_frac, _ = CONFIGS[cfg_name]
    if family == "mlp":
        m = lcb.make_base_model(3072, classes, C1_WIDTHS, 8, seed)
        vs = [lcb.build_variant(l + 1, l, C1_MENU[l], m.tap_dim(l + 1), classes, seed + 1) for l in range(8)]
        calib = mlp_inputs(min(max(batch, 128), 512), 3072, seed + 2)
        gen = lambda B, s: mlp_inputs(B, 3072, s)  # noqa: E731
    else:
        m = lcb.make_cnn_model(arch, classes, seed)
        vs = []
        for l in range(1, m.num_blocks + 1):
            C, H, W = m.tap(l)
            # C4 (VGG-16): FC and pool cache models on alternate taps; else Pool(C) = GAP heads
            a = ("FC(256)" if l % 2 == 0 else f"Pool({C})") if arch.startswith("vgg") else f"Pool({C})"
            vs.append(lcb.build_variant(l, 0, a, m.tap_dim(l), classes, seed + l))
        side = 32 if arch.endswith("cifar") else 224
        calib = image_inputs(min(max(batch, 128), 256), 3, side, side, seed + 2)  # >= 128 images even at batch 1
        gen = lambda B, s: image_inputs(B, 3, side, side, s)  # noqa: E731
    fr = calibrate_variants(m, vs, calib, full_frac, precision=precision, device=device)
    dep = lcb.Deployment(m, vs, precision=precision, max_batch=batch, device=device)
    base = lcb.Deployment(m, [], precision=precision, max_batch=batch, device=device)
    return m, vs, dep, base, gen, fr


C1_WIDTHS = [64, 64, 128, 128, 256, 256, 512, 512]  # = paper_2101_07344_b200.synthetic.C1_WIDTHS
C1_MENU = ["FC(1024)", "Pool(8192)", "Conv(3,1)", "FC(512)", "Pool(4096)", "Conv(5,2)", "FC(1024)", "Pool(8192)"]


def cpu_reference(cfg_name, steps, warmup, seed=2101):
    """The reference's CPU path on this host's cores (bounded sample per step).

    Never imports or loads the product library: the block-MLP config runs the
    reference's own make_base_model / build_variant / simulate_model
    (oracle/_ref, the unmodified reference compiled from its sources); the
    CNN configs (no reference counterpart) build the same synthetic network
    with oracle/cnn_models.py (bit-identical weights to make_cnn_model, pinned
    by tests/test_oracle.py), run its fp64 forward through the C restatement
    (oracle/lc_oracle.c) and every cache lookup through the reference's own
    lookup() (oracle/_ref; the restatement when _ref is absent)."""
    from oracle import oracle as O
    family, arch, classes, _, _, _ = CONFIGS[cfg_name]
    cores = os.cpu_count() or 1
    have_ref = os.path.exists(O.REF_SO)
    if family == "mlp":
        rm = O.RefModel.make(3072, classes, C1_WIDTHS, 8, seed)
        rvs = [O.RefVariant.build(l + 1, l, C1_MENU[l], rm.tap_dims[l], classes, seed + 1) for l in range(8)]
        sample = 4096
        x = np.random.default_rng(seed + 3).uniform(-1.5, 1.5, size=(sample, 3072))
        kind = "reference"
        run = lambda: O.ref_simulate(rm, rvs, x, threads=cores)  # noqa: E731
        desc = f"{sample} requests of the C1 block-MLP through the reference's simulate_model (oracle/_ref), " \
               f"request-sharded over {cores} threads"
    else:
        from oracle.cnn_models import CnnModel
        cm = CnnModel(arch, classes, seed)
        side = cm.in_shape[1]
        sample = max(2 * cores, 16) if arch.endswith("cifar") else max(cores // 2, 4)
        x = np.random.default_rng(seed + 3).standard_normal((sample, 3 * side * side))
        if have_ref:
            vs = [O.RefVariant.build(l, 0, f"Pool({cm.taps[l - 1][0]})", cm.tap_dims[l - 1], classes, seed + l)
                  for l in range(1, cm.num_blocks + 1)]
            look = lambda k, t: vs[k].lookup(t, classes)[0]  # noqa: E731
        else:
            raise RuntimeError("oracle/_ref (the compiled reference) is required for the reference arm")
        kind = "port"

        def run():
            taps, _ = O.oracle_cnn_forward(cm.ops, cm.nslots, x, cm.num_blocks, cm.tap_dims, classes, threads=cores)
            for i in range(sample):
                for k in range(cm.num_blocks):
                    if look(k, taps[k][i]):
                        break
        desc = f"{sample} images per step: fp64 forward of {arch} through the C restatement (oracle/lc_oracle.c, " \
               f"image-sharded over {cores} threads; the reference has no CNN) + the reference's own lookup() " \
               f"(oracle/_ref) per cache until the first hit"
    for _ in range(max(0, warmup)):
        run()
    t0 = time.perf_counter()
    for _ in range(steps):
        run()
    dt = time.perf_counter() - t0
    out = {"value": sample * steps / dt, "unit": "requests/s", "cores": cores, "kind": kind, "sample": desc}
    if family == "mlp":
        # the reference on one core as well (a 1024-request sample)
        x1 = x[:1024]
        O.ref_simulate(rm, rvs, x1[:64], threads=1)
        t0 = time.perf_counter()
        O.ref_simulate(rm, rvs, x1, threads=1)
        out["single_core"] = {"value": len(x1) / (time.perf_counter() - t0), "unit": "requests/s", "cores": 1,
                              "sample": "1024 requests of the same workload, one thread"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50", choices=sorted(CONFIGS))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--precision", default="bf16x3", choices=["bf16x3", "bf16"])
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--sweep", default="",
                    help="comma-separated thresholds: C4 confidence-threshold sweep (req/s, hit rate and agreement "
                         "with the base model per threshold) instead of the single-threshold line")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "timing rules: at least 3 warm-up steps"

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    family, arch, classes, dflt_batch, full_frac, cfg_str = CONFIGS[args.config]
    B = args.batch or dflt_batch
    metric = "requests/sec with learned caches (p50/p99 latency, no-cache req/s, hit rate alongside)"
    config = {"workload": args.config, "baseline_config": cfg_str, "batch_per_gpu": B, "global_batch": B * world,
              "caches": ("FC(256) / Pool(C) heads on alternate pool-stage taps + FC(16) selector"
                         if arch and arch.startswith("vgg") else "Pool(C) GAP head + FC(16) selector after every block")
              if family == "cnn" else "one build_variant cache per block (FC/Pool/Conv menu)",
              "exit_profile_full_fraction": full_frac, "precision": args.precision,
              "l2": "flushed (256 MiB write) between timed steps, outside the events",
              "parallelism": f"dp{world} (request shards, no collectives)"}

    if args.impl == "reference":
        if rank != 0:
            return
        cb = cpu_reference(args.config, args.steps, args.warmup)
        try:  # evidence that this arm ran without the product library
            maps = open("/proc/self/maps").read()
            cb["product_library_loaded"] = "liblatecache_b200" in maps
            cb["reference_library_loaded"] = "liblatecache_ref" in maps
        except OSError:
            pass
        line = {"metric": metric, "value": cb["value"], "unit": "requests/s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "impl": "reference", "cpu_baseline": cb,
                "e2e": {"value": cb["value"], "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2101_07344_b200 as lcb

    m, vs, dep, base, gen, fractions = build_deployment(args.config, B, args.precision, local)
    nbatches = 4
    inputs = [gen(B, 1000 + rank * 101 + j).astype(np.float32) for j in range(nbatches)]
    dev_inputs = [torch.from_numpy(x).cuda() for x in inputs]
    pinned = [torch.from_numpy(x).pin_memory() for x in inputs]
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    in_ptr, base_ptr = dep, base

    def stage(d, j):
        # step j's inputs are already resident in HBM; D2D into the engine's input buffer
        torch.cuda.synchronize()
        d.stage_input_device(dev_inputs[j].data_ptr(), B)

    def run_steps(d, ptr, steps, collect):
        total_ms = 0.0
        lats, exits = [], []
        for s in range(steps):
            j = s % nbatches
            stage(ptr, j)
            flush.zero_()
            torch.cuda.synchronize()
            total_ms += d.serve_timed(B)
            if collect:
                r = d.results(B)
                lats.append(r.latency_ms.copy())
                exits.append(r.exit_layer.copy())
        return total_ms, lats, exits

    if args.sweep:
        rows = []
        for d in [float(t) for t in args.sweep.split(",")]:
            for v in vs:
                dep.set_delta(v.layer, d)
            run_steps(dep, in_ptr, args.warmup, False)
            ms, lats, exits = run_steps(dep, in_ptr, args.steps, True)
            sh = dep.serve(inputs[0], shadow=True)
            ex = np.concatenate(exits)
            lat = np.concatenate(lats)
            hit = sh.exit_layer > 0
            rows.append({"delta": d, "requests_per_s": B * args.steps * world / (ms / 1e3),
                         "ms_per_step": ms / args.steps, "hit_rate": float(np.mean(ex > 0)),
                         "p50_ms": float(lcb.nearest_rank(lat, 0.5)), "p99_ms": float(lcb.nearest_rank(lat, 0.99)),
                         "agreement_with_base": float(np.mean(sh.served == sh.base_pred)),
                         "hit_accuracy": float(np.mean(sh.served[hit] == sh.base_pred[hit])) if hit.any() else 1.0})
        line = {"metric": "requests/sec vs confidence threshold (C4 sweep; hit rate, agreement with the base model)",
                "value": rows[0]["requests_per_s"], "unit": "requests/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "bf16x3 (hi/lo bf16 split, fp32 accumulate: fp32-class)" if args.precision == "bf16x3"
                else "bf16", "data": "synthetic", "config": dict(config, sweep=args.sweep), "sweep": rows}
        if rank == 0:
            print(json.dumps(line))
        if dist:
            dist.destroy_process_group()
        return

    # warm-up (graph capture happens here)
    run_steps(dep, in_ptr, args.warmup, False)
    run_steps(base, base_ptr, args.warmup, False)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    barrier()
    with ClockSampler(local) as clk:
        ms_cache, lats, exits = run_steps(dep, in_ptr, args.steps, True)
    barrier()
    ms_base, base_lats, _ = run_steps(base, base_ptr, args.steps, True)
    barrier()

    # e2e through the public API from pinned host buffers (H2D + serve + D2H of
    # every step in the region), pipelined two deep: submit(i + 1) uploads while
    # batch i computes; collect(i) returns its results to the host.
    for s in range(args.warmup):  # pipeline set-up (slot buffers, copy stream) outside the region
        dep.collect(dep.submit(pinned[s % nbatches].numpy()))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pending = []
    for s in range(args.steps):
        pending.append(dep.submit(pinned[s % nbatches].numpy()))
        if len(pending) == 2:
            dep.collect(pending.pop(0))
    while pending:
        dep.collect(pending.pop(0))
    e2e_s = time.perf_counter() - t0
    barrier()

    from paper_2101_07344_b200.shard import max_over_ranks as _mor

    def max_over_ranks(v):
        return _mor(v, dist, device="cuda")

    ms_cache_max = max_over_ranks(ms_cache)
    ms_base_max = max_over_ranks(ms_base)
    e2e_max = max_over_ranks(e2e_s)
    total_req = B * args.steps * world
    value = total_req / (ms_cache_max / 1e3)
    lat = np.concatenate(lats)
    blat = np.concatenate(base_lats)
    ex = np.concatenate(exits)
    hit_rate = float(np.mean(ex > 0))
    hits_by_layer = {int(l): int(np.sum(ex == l)) for l in range(1, m.num_blocks + 1) if np.sum(ex == l)}

    # Roofline of the dominant kernels (the tcgen05 contractions), measured live.
    # The graphed, timed step has no per-kernel events, so each kind's share of
    # the step comes from one un-graphed batch with CUDA events around every
    # launch (same step list, same survivors), applied to the timed graphed
    # step: kernel ms per step = ms_per_step x share <= ms_per_step.
    stage(dep, 0)
    prof = dep.profile(B)
    step_ms = float(prof["ms"].sum())
    ms_step = ms_cache_max / args.steps

    def kind_share(mask):
        return float(prof["ms"][mask].sum()) / step_ms if step_ms else 0.0

    tc = prof["kind"] == 1
    lk = prof["kind"] == 2
    glue = prof["kind"] == 0
    tc_flops = float(prof["flops"][tc].sum())
    tc_bytes = float(prof["bytes"][tc].sum())
    tc_ms = ms_step * kind_share(tc)
    lk_ms = ms_step * kind_share(lk)
    lk_bytes = float(prof["bytes"][lk].sum())
    glue_ms = ms_step * kind_share(glue)
    glue_bytes = float(prof["bytes"][glue].sum())
    hbm, bf16_burst, bf16_sus, peak_src = load_peaks()
    mma_factor = 3.0 if args.precision == "bf16x3" else 1.0
    # Per contraction launch: tensor floor (MMA FLOPs at the bf16 peak) and HBM
    # floor (algorithmic bytes: input + output + residual once, at the copy
    # bandwidth); the binding floor summed over launches / their measured time
    # is the combined roofline fraction (from the un-graphed per-launch events).
    t_tc = prof["flops"][tc] * mma_factor / (bf16_burst * 1e12) * 1e3
    t_hbm = prof["bytes"][tc] / (hbm * 1e9) * 1e3
    floor_ms = float(np.maximum(t_tc, t_hbm).sum())
    bound = "tensor" if float(t_tc.sum()) >= float(t_hbm.sum()) else "hbm"
    ach_tf = tc_flops / (tc_ms * 1e-3) / 1e12 if tc_ms else 0.0
    ach_gb = tc_bytes / (tc_ms * 1e-3) / 1e9 if tc_ms else 0.0
    traffic = traffic_src = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.precision}.json")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        traffic, traffic_src = tj.get("dram_bytes_per_step"), tj.get("source")
    roofline = {"bound": bound, "kernel": "tc_conv_kernel + tc_stem_kernel (tcgen05 implicit-GEMM convs)",
                "achieved": ach_tf if bound == "tensor" else ach_gb,
                "peak": bf16_burst if bound == "tensor" else hbm,
                "unit": "TFLOP/s" if bound == "tensor" else "GB/s",
                "frac": (ach_tf / bf16_burst) if bound == "tensor" else ach_gb / hbm,
                "traffic": traffic, "traffic_source": traffic_src, "algorithmic_bytes_per_step": tc_bytes,
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json: bf16 burst {bf16_burst} TFLOP/s, HBM {hbm} GB/s)",
                "algorithmic_flops_per_step": tc_flops, "kernel_ms_per_step": tc_ms, "ms_per_step": ms_step,
                "share_of_step": kind_share(tc),
                "mma_flops_per_algorithmic_flop": mma_factor,
                "tensor_pipe_issue_frac": ach_tf * mma_factor / bf16_burst, "hbm_frac": ach_gb / hbm,
                "combined_floor_ms_per_step": floor_ms,
                "combined_frac": floor_ms / float(prof["ms"][tc].sum()) if tc.any() else None,
                "definition": "achieved = algorithmic FLOPs (2 x MACs executed on the surviving requests) / the "
                              "contractions' time inside the timed graphed step (ms_per_step x their share of an "
                              "un-graphed event-timed step); frac = achieved / peak. tensor_pipe_issue_frac counts "
                              "the MMA FLOPs issued (x3 in bf16x3). combined_frac = sum of per-launch "
                              "max(tensor floor, HBM floor) / sum of per-launch event times"}
    roofline_lookup = {"bound": "latency (per-row heads over L2-resident GAP partials; HBM bytes are negligible)",
                       "achieved": lk_bytes / (lk_ms * 1e-3) / 1e9 if lk_ms else 0.0,
                       "peak": hbm, "unit": "GB/s",
                       "frac": (lk_bytes / (lk_ms * 1e-3) / 1e9 / hbm) if lk_ms else 0.0,
                       "kernel_ms_per_step": lk_ms, "share_of_step": kind_share(lk)}
    roofline_glue = {"bound": "hbm", "kernels": "stem space-to-depth, max-pool, base head, batch init",
                     "algorithmic_bytes_per_step": glue_bytes, "kernel_ms_per_step": glue_ms,
                     "achieved": glue_bytes / (glue_ms * 1e-3) / 1e9 if glue_ms else 0.0, "peak": hbm, "unit": "GB/s",
                     "frac": glue_bytes / (glue_ms * 1e-3) / 1e9 / hbm if glue_ms else 0.0,
                     "share_of_step": kind_share(glue)}

    line = {
        "metric": metric, "value": value, "unit": "requests/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_cache_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16x3 (hi/lo bf16 split, fp32 accumulate: fp32-class)" if args.precision == "bf16x3" else "bf16",
        "data": "synthetic (seeded N(0,1) images / uniform vectors; random-init weights, calibrated selectors)",
        "config": config,
        "latency_ms": {"p50": float(lcb.nearest_rank(lat, 0.5)), "p99": float(lcb.nearest_rank(lat, 0.99)),
                       "definition": "device time from batch start to the request's exit (nearest-rank)"},
        "no_cache": {"value": total_req / (ms_base_max / 1e3), "unit": "requests/s",
                     "ms_per_step": ms_base_max / args.steps,
                     "p50_ms": float(lcb.nearest_rank(blat, 0.5)), "p99_ms": float(lcb.nearest_rank(blat, 0.99))},
        "speedup_vs_no_cache": ms_base_max / ms_cache_max,
        "hit_rate": hit_rate, "hits_by_layer": hits_by_layer,
        "e2e": {"value": total_req / e2e_max, "unit": "requests/s",
                "h2d_bytes_per_step": int(inputs[0].nbytes),
                "d2h_bytes_per_step": int(B * (4 * 3 + 8) + B * m.num_blocks * 4 + B * m.num_classes * 4 + 8)},
        "gpu_launches": dep.kernel_count() * args.steps,
        "roofline": roofline, "roofline_lookup": roofline_lookup, "roofline_glue": roofline_glue,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_reference(args.config, args.cpu_steps, 1)
    if rank == 0:
        print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
