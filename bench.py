#!/usr/bin/env python
"""Benchmark of the learned-cache serve path (BASELINE.json metric: requests/s
and p50/p99 latency with learned caches vs no-cache; hit rate).

Default workload = BASELINE.json configs[1]: ResNet-18 CIFAR-10 shape with a
learned cache (Pool(C) = GAP head + selector) after every residual block,
batch 256 per GPU, synthetic weights and N(0,1) images, selectors calibrated
to the paper's R18-C10 exit profile (3.51 % of requests run the full model,
PAPER.md:2873-2878). One step = one batch through the serve path on every GPU.

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


def cpu_reference(cfg_name, steps, warmup, seed=2101):
    """The reference's CPU path on this host's cores (bounded sample per step)."""
    from oracle import oracle as O
    import paper_2101_07344_b200 as lcb
    from paper_2101_07344_b200.synthetic import C1_MENU, C1_WIDTHS, image_inputs, mlp_inputs
    family, arch, classes, _, _, _ = CONFIGS[cfg_name]
    cores = os.cpu_count() or 1
    if family == "mlp":
        rm = O.RefModel.make(3072, classes, C1_WIDTHS, 8, seed)
        rvs = [O.RefVariant.build(l + 1, l, C1_MENU[l], rm.tap_dims[l], classes, seed + 1) for l in range(8)]
        sample = 4096
        x = mlp_inputs(sample, 3072, seed + 3)
        kind = "reference"
        run = lambda: O.ref_simulate(rm, rvs, x, threads=cores)  # noqa: E731
        desc = f"{sample} requests of the C1 block-MLP through the reference's simulate_model (oracle/_ref), " \
               f"request-sharded over {cores} threads"
    else:
        m = lcb.make_cnn_model(arch, classes, seed)
        ops = m.cnn_ops()
        side = 32 if arch.endswith("cifar") else 224
        sample = max(2 * cores, 16) if arch.endswith("cifar") else max(cores // 2, 4)
        x = image_inputs(sample, 3, side, side, seed + 3)
        vs = []
        for l in range(1, m.num_blocks + 1):
            C, H, W = m.tap(l)
            v = lcb.build_variant(l, 0, f"Pool({C})", m.tap_dim(l), classes, seed + l)
            pred, sel, d = O.variant_layers_from_product(v)
            vs.append((O.OracleNet(pred), O.OracleNet(sel), d))
        kind = "port"

        def run():
            taps, logits = O.oracle_cnn_forward(ops, m.nslots, x, m.num_blocks, m.tap_dims, classes, threads=cores)
            for i in range(sample):
                for l, (pn, sn, d) in enumerate(vs):
                    if O.oracle_lookup(pn, sn, d, taps[l][i])[0]:
                        break
        desc = f"{sample} images per step through the fp64 C restatement of {arch} (oracle/lc_oracle.c) + " \
               f"the reference lookup restatement, image-sharded over {cores} threads (the reference has no CNN)"
    for _ in range(max(0, warmup)):
        run()
    t0 = time.perf_counter()
    for _ in range(steps):
        run()
    dt = time.perf_counter() - t0
    return {"value": sample * steps / dt, "unit": "requests/s", "cores": cores, "kind": kind, "sample": desc}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet18_cifar", choices=sorted(CONFIGS))
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

    # live roofline: per-step CUDA events over one (un-graphed) batch
    stage(dep, 0)
    prof = dep.profile(B)
    tc = prof["kind"] == 1
    tc_ms = float(prof["ms"][tc].sum())
    tc_flops = float(prof["flops"][tc].sum())
    tc_bytes = float(prof["bytes"][tc].sum())
    lk = prof["kind"] == 2
    lk_ms = float(prof["ms"][lk].sum())
    lk_bytes = float(prof["bytes"][lk].sum())
    step_ms = float(prof["ms"].sum())
    hbm, bf16_burst, bf16_sus, peak_src = load_peaks()
    mma_factor = 3.0 if args.precision == "bf16x3" else 1.0
    # Per contraction launch: tensor floor (MMA FLOPs at the bf16 peak) and HBM
    # floor (algorithmic bytes: input + output + residual once, at the copy
    # bandwidth); the binding floor summed over launches / their measured time
    # is the combined roofline fraction.
    t_tc = prof["flops"][tc] * mma_factor / (bf16_burst * 1e12) * 1e3
    t_hbm = prof["bytes"][tc] / (hbm * 1e9) * 1e3
    floor_ms = float(np.maximum(t_tc, t_hbm).sum())
    bound = "tensor" if float(t_tc.sum()) >= float(t_hbm.sum()) else "hbm"
    ach_tf = tc_flops / (tc_ms * 1e-3) / 1e12 if tc_ms else 0.0
    ach_gb = tc_bytes / (tc_ms * 1e-3) / 1e9 if tc_ms else 0.0
    traffic = None
    tpath = os.path.join(ROOT, "profiles", f"traffic_{args.config}_{args.precision}.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get("dram_bytes_per_step")
    roofline = {"bound": bound, "kernel": "tc_conv_kernel + tc_stem_kernel (tcgen05 implicit-GEMM convs)",
                "achieved": ach_tf if bound == "tensor" else ach_gb,
                "peak": bf16_burst if bound == "tensor" else hbm,
                "unit": "TFLOP/s" if bound == "tensor" else "GB/s",
                "frac": (ach_tf * mma_factor / bf16_burst) if bound == "tensor" else ach_gb / hbm,
                "traffic": traffic, "algorithmic_bytes_per_step": tc_bytes,
                "peak_source": f"{peak_src} (MEASURED_PEAKS.json: bf16 burst {bf16_burst} TFLOP/s, HBM {hbm} GB/s)",
                "algorithmic_flops_per_step": tc_flops, "kernel_ms_per_step": tc_ms,
                "share_of_step": tc_ms / step_ms if step_ms else None,
                "mma_flops_per_algorithmic_flop": mma_factor,
                "tensor_pipe_frac": ach_tf * mma_factor / bf16_burst, "hbm_frac": ach_gb / hbm,
                "combined_floor_ms_per_step": floor_ms,
                "combined_frac": floor_ms / tc_ms if tc_ms else None,
                "definition": "per launch floor = max(MMA FLOPs / bf16 peak, algorithmic bytes / HBM peak); "
                              "combined_frac = sum of floors / sum of measured launch times (CUDA events, "
                              "one un-graphed batch)"}
    roofline_lookup = {"bound": "latency (per-row heads over L2-resident GAP partials; HBM bytes are negligible)",
                       "achieved": lk_bytes / (lk_ms * 1e-3) / 1e9 if lk_ms else 0.0,
                       "peak": hbm, "unit": "GB/s",
                       "frac": (lk_bytes / (lk_ms * 1e-3) / 1e9 / hbm) if lk_ms else 0.0,
                       "kernel_ms_per_step": lk_ms, "share_of_step": lk_ms / step_ms if step_ms else None}

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
                "d2h_bytes_per_step": int(B * (4 * 3 + 8) + B * m.num_blocks * 4)},
        "gpu_launches": dep.kernel_count() * args.steps,
        "roofline": roofline, "roofline_lookup": roofline_lookup,
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
