#!/usr/bin/env python
"""bench.py — requests bucketed+packed per second on B200 (BASELINE.json metric).

One step = one window of the BucketServe scheduling hot path over a fresh-in-HBM
synthetic window: K1 histogram -> [C1 NCCL histogram all-reduce when N>1] -> K2
boundaries -> K3/K4 assign+order -> K5 size -> K6 pack (padded [n, pitch] int32
tokens + u8 mask).  Default workload = BASELINE configs[1] (C2): 1M requests per
GPU, lognormal ShareGPT-like lengths, Llama-2-7B KV model on 180 GiB / 14 GiB.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c3|c4]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one rank per GPU)
    python bench.py --impl reference ...                      (CPU reference arm)

Prints ONE JSON line on rank 0.  `value` is device-timed (CUDA events, max over
ranks) with inputs resident in HBM; `e2e` is the same metric through the public
API from pinned HOST buffers with the H2D of every input and the D2H of the
schedule inside the timed region.  Inputs (1.75 GB token store per GPU) exceed the
126 MB L2, so no explicit flush is needed between steps.
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

METRIC = "requests bucketed+packed/sec"
UNIT = "requests/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _pack_kernel(l_max, max_n, n_classes=1, dispatch=False, world=1):
    """the K6 kernel(s) the library launches by default (k_pack.cu: launch_pack); windows
    K0 takes (k_small.cu: small_window_ok — <= 2048 requests, l_max <= 8192, one rank, no
    dispatch order) are copied by k_pack_rows."""
    if (os.environ.get("BS_SMALL", "1") != "0" and not dispatch and world == 1
            and max_n <= 2048 and l_max <= 8192 and l_max * n_classes <= 16384):
        return "k_pack_rows"
    v = int(os.environ.get("BS_PACK_VARIANT", "0") or 0)
    if v not in (1, 5, 21):
        v = 1
    return {1: "k_pack_bulk", 5: "k_pack_tma", 21: "k_pack_stream"}[v]


def _profile_traffic(cfg_name, kernel):
    """dram bytes per pack launch from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        ent = d.get(kernel, {}).get(cfg_name)
        return ent.get("dram_bytes") if ent else None
    except Exception:
        return None


_ALL_CPUS = None


def _bind_near_gpu(index):
    """Run this rank on the CPU cores NVML reports as local to its GPU (the socket whose
    PCIe root holds it), so the pinned host buffers of the e2e leg are allocated on that
    NUMA node; returns the core count, or None when NVML cannot tell."""
    global _ALL_CPUS
    _ALL_CPUS = os.sched_getaffinity(0)
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 50 ms during the timed region."""

    FIELDS = ("clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", str(self.index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = set()
        names = ("sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")
        for r in self.rows:
            for nm, v in zip(names, r[3:]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def cpu_port_window(cfg, lens, cls, tok_off, tokens, threads, out_capacity=None):
    from oracle import cpu
    ws = cpu.WindowSpec(l_max=cfg.l_max, n_classes=cfg.n_classes, policies=cfg.policies,
                        theta=cfg.theta, adjust=cfg.adjust, kvpt=cfg.kvpt,
                        current_safe=cfg.current_safe, accounting=cfg.accounting,
                        init_edges=cfg.init_edges)
    return cpu.window(ws, lens, cls, tok_off, tokens, threads=threads, out_capacity=out_capacity)


def cpu_baseline(cfg_name, n_sample, budget_s=12.0):
    """The oracle port (oracle/bso.c, all host threads) on bounded C2-shaped windows."""
    from paper_2507_17120_b200 import workloads as W
    cfg, lens, cls = W.make_window(cfg_name, n=n_sample, seed=99)
    tok_off, tokens = W.token_store(lens)
    threads = os.cpu_count() or 1
    r = cpu_port_window(cfg, lens, cls, tok_off, tokens, threads)
    cap = int(r.summary["packed_elems"])
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        cpu_port_window(cfg, lens, cls, tok_off, tokens, threads, out_capacity=cap)
        times.append(time.perf_counter() - t0)
        if len(times) >= 50:
            break
    med = statistics.median(times)
    return {"value": n_sample / med, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{cfg_name} distribution, {n_sample}-request windows incl. pack, "
                      f"{len(times)} runs, median {med:.3f} s (oracle/bso.c, OpenMP)"}


def run_reference(args, rank, world):
    """--impl reference: the reference path's CPU implementation (oracle port) on the
    same config / metric, rank 0 only."""
    if rank != 0:
        return
    from paper_2507_17120_b200 import workloads as W
    # the same window as the B200 arm (one full config-sized window per step) unless a
    # smaller --cpu-sample is forced, which the line then reports as same_config: false
    n_ref = args.requests if args.cpu_sample is None else min(args.requests, args.cpu_sample)
    cfg, lens, cls = W.make_window(args.config, n=n_ref, seed=1234)
    tok_off, tokens = W.token_store(lens)
    threads = os.cpu_count() or 1
    r = cpu_port_window(cfg, lens, cls, tok_off, tokens, threads)
    cap = int(r.summary["packed_elems"])
    for _ in range(args.warmup):
        cpu_port_window(cfg, lens, cls, tok_off, tokens, threads, out_capacity=cap)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_port_window(cfg, lens, cls, tok_off, tokens, threads, out_capacity=cap)
    dt = (time.perf_counter() - t0) / args.steps
    value = len(lens) / dt
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (seeded lengths, hashed token ids)", "impl": "reference",
        "config": {"workload": f"{args.config}: {cfg.note}", "requests_per_step": len(lens),
                   "parallelism": "host threads", "same_config": len(lens) == args.requests},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.config} distribution, {len(lens)}-request window per "
                                   "step incl. pack (reference composition restated in C, "
                                   "oracle/bso.c, OpenMP)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not args.no_reference_python:
        line["reference_python"] = reference_python_leg(args, lens, cls, cfg)
    print(json.dumps(line), flush=True)


def reference_python_leg(args, lens, cls, cfg):
    """The UNMODIFIED reference itself (bucketsim's classes composed as SURVEY §3.4,
    oracle/ref_compose.py) timed on this host, one thread pinned to one core, on the
    arm's window (or a --ref-python-sample-request window of the config), checked
    against the oracle port: tools/ref_python_bench.py in a child process (the pin stays
    out of this process).  Needs the reference package: /root/reference, or its pip
    install in baseline/_ref (made by __graft_entry__.build()).  Reported beside the
    port, not as the line's value."""
    n = min(len(lens), args.ref_python_sample)
    cmd = [sys.executable, os.path.join(ROOT, "tools", "ref_python_bench.py"),
           "--window", f"{args.config}:{n}"]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=900,
                           env=dict(os.environ, OMP_NUM_THREADS="1"))
        ln = [x for x in r.stdout.splitlines() if x.startswith("{")]
        if not ln:
            return {"unavailable": (r.stderr or "no output").strip().splitlines()[-1][-300:]}
        d = json.loads(ln[-1])
    except subprocess.TimeoutExpired:
        return {"unavailable": "timed out after 900 s"}
    return {"value": d["requests_per_s"], "unit": UNIT, "cores": 1, "seconds": d["seconds"],
            "requests": d["requests"], "batches": d["batches"], "nproc": d["nproc"],
            "oracle_parity": d["oracle_parity"],
            "kind": "reference (bucketsim, unmodified, pure Python)",
            "sample": f"{args.config} window of {n} requests (seed 1234: the arm's own window "
                      f"when {n} = {len(lens)}), one run (assign, adjust_buckets fixpoint, "
                      "form_batch drain), checked against the oracle port"}


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _spawn_ranks(args):
    """`--gpus N` without a launcher: re-run this script as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1.  More ranks than visible GPUs only with
    --share-gpus (gloo process group, ranks share GPUs round-robin, collective 'torch'
    or 'peer'); otherwise a one-line JSON refusal."""
    import torch
    n_dev = torch.cuda.device_count()
    env = dict(os.environ)
    argv = list(sys.argv[1:])
    if args.gpus > n_dev:
        if not args.share_gpus:
            print(json.dumps({"metric": METRIC, "impl": args.impl, "n_gpus": args.gpus,
                              "unavailable": f"{args.gpus} GPUs requested, {n_dev} visible; "
                                             "pass --share-gpus to run the ranks on the visible "
                                             "GPUs (gloo, functional check only)"}), flush=True)
            return
        env["BS_DIST_BACKEND"] = "gloo"
        if args.collective == "nccl":  # NCCL needs one GPU per rank
            argv += ["--collective", "torch"]
    if args.gpus > 1 and args.impl == "b200":
        env.setdefault("NCCL_DEBUG", "INFO")           # communicator lines on stderr
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + argv
    rc = subprocess.call(cmd, env=env)
    if rc:
        sys.exit(rc)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--requests", type=int, default=None, help="requests per GPU (default: config)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reference-python", action="store_true", help="--impl reference: "
                    "skip timing the unmodified Python reference beside the port")
    ap.add_argument("--ref-python-sample", type=int, default=1_000_000, help="requests of the "
                    "window the unmodified Python reference is timed on (one run)")
    ap.add_argument("--no-graph", action="store_true", help="launch the window kernels "
                    "individually instead of replaying one CUDA graph per window")
    ap.add_argument("--cpu-sample", type=int, default=None, help="requests per window of the "
                    "CPU arms (default: the full window for --impl reference, 131,072 for the "
                    "cpu_baseline leg of the B200 line)")
    ap.add_argument("--share-gpus", action="store_true", help="with --gpus N larger than the "
                    "visible GPUs: run the N ranks on the visible ones (gloo process group, "
                    "collective 'torch') instead of refusing")
    ap.add_argument("--dispatch", action="store_true", help="also compute the simulator's "
                    "global dispatch order (K7, SURVEY f3) inside every window")
    ap.add_argument("--collective", default="nccl", choices=["nccl", "torch", "peer"],
                    help="C1 for N > 1: 'nccl' = the library's own NCCL communicator, the "
                         "histogram all-reduce issued between K1 and K2 inside the window's CUDA "
                         "graph (NVLink / NVSwitch); 'torch' = torch.distributed.all_reduce "
                         "between an eager K1 and the graph of K2..K6; 'peer' = device-side "
                         "exchange over CUDA-IPC peer memory (bs_peer_*)")
    ap.add_argument("--inflight", type=int, default=0, help="windows in flight: consecutive "
                    "windows alternate over this many schedulers (own scratch, outputs and CUDA "
                    "stream), so the latency-bound scheduling of one window overlaps the "
                    "HBM-bound pack of the previous ones; 0 = as many as HBM holds, up to 4")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _spawn_ranks(args)
        return

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_2507_17120_b200 import workloads as W
    cfg0 = W.CONFIGS[args.config]
    if args.requests is None:
        args.requests = cfg0.n // world if args.config == "c5" else cfg0.n

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.config == "c5" and world < 2 and args.requests > 32_000_000:
        # 64M requests: ~115 GB of token store + ~145 GB of packed output on one GPU
        print(json.dumps({"metric": METRIC, "impl": "b200", "config": {"workload": "c5"},
                          "unavailable": "C5 (64M requests) is sharded over >= 2 GPUs; pass "
                                         "--requests to run a smaller window on one"}), flush=True)
        return

    import torch
    import torch.distributed as dist
    # one process per GPU; ranks beyond the visible GPUs share them round-robin (lets the
    # distributed path run on a one-GPU box with BS_DIST_BACKEND=gloo)
    local_dev = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    numa_cpus = _bind_near_gpu(local_dev)
    pg = None
    if world > 1:
        backend = os.environ.get("BS_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist.group.WORLD
    from paper_2507_17120_b200.window import WindowScheduler

    if args.config == "c5":  # one 64M-request trace, contiguous arrival-order shard per rank
        cfg, lens_np, cls_np = W.make_window("c5", n=args.requests * world, seed=1234,
                                             shard=(rank, world))
    else:
        cfg, lens_np, cls_np = W.make_window(args.config, n=args.requests, seed=1234 + rank)
    n = len(lens_np)
    lens = torch.as_tensor(lens_np).to(dev)
    cls = torch.as_tensor(cls_np).to(dev)
    tok_off, tokens = W.token_store_device(lens, seed=rank)
    torch.cuda.synchronize(dev)
    free0 = torch.cuda.mem_get_info(dev)[0]

    def make_sched():
        return WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                               policies=cfg.policies, split_threshold=cfg.theta,
                               adjust=cfg.adjust, buckets=cfg.init_edges,
                               kv_bytes_per_token=cfg.kvpt, current_safe=cfg.current_safe,
                               accounting=cfg.accounting, device=dev, process_group=pg,
                               dispatch=args.dispatch, collective=args.collective)

    # first window sizes the reusable packed-output buffer.  If the library's own NCCL
    # communicator cannot be set up on some rank (e.g. libnccl not resolvable), every rank
    # falls back to torch.distributed's all-reduce between K1 and K2, and the line says so
    fallback = None
    try:
        sched = make_sched()
        res = sched.schedule(lens, cls, tok_off, tokens)
        failed = 0
    except Exception as err:  # noqa: BLE001 - reported in the line, then retried
        failed, fallback = 1, f"collective {args.collective} failed ({type(err).__name__}: {err})"
    if pg is not None and args.collective == "nccl":
        flag = torch.tensor([failed], device=dev)
        dist.all_reduce(flag)
        if int(flag.item()) and args.collective != "torch":
            fallback = fallback or "collective nccl failed on another rank"
            args.collective = "torch"
            print(f"bench: {fallback}; using collective torch", file=sys.stderr, flush=True)
            sched = make_sched()
            res = sched.schedule(lens, cls, tok_off, tokens)
    elif failed:
        raise RuntimeError(fallback)
    s0 = res.summary()
    l_b = sched.ctx.launches
    res = sched.schedule(lens, cls, tok_off, tokens)
    kernels_per_window = sched.ctx.launches - l_b
    use_graph = not args.no_graph
    # stage breakdown: a separate profiled pass (events between the kernels of the
    # eager launch sequence), not part of the timed region
    for _ in range(2):
        sched.schedule(lens, cls, tok_off, tokens, sync=False, check=False)
    sched.ctx.profile_enable(args.steps)
    for _ in range(args.steps):
        sched.schedule(lens, cls, tok_off, tokens, sync=False, check=False)
    torch.cuda.synchronize(dev)
    stage_ms, prof_steps = sched.ctx.profile_read()
    stage_ms = {k: v / max(prof_steps, 1) for k, v in stage_ms.items()}
    sched.ctx.profile_enable(0)
    c1_ms = stage_ms.get("exchange", 0.0) if world > 1 else None
    if world > 1 and args.collective == "torch":  # C1 outside the library: time it here
        from paper_2507_17120_b200.sharding import allreduce_histogram
        for _ in range(3):
            allreduce_histogram(sched.hist_global, pg)
        e_a, e_b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e_a.record()
        for _ in range(20):
            allreduce_histogram(sched.hist_global, pg)
        e_b.record()
        torch.cuda.synchronize(dev)
        c1_ms = e_a.elapsed_time(e_b) / 20
    # windows in flight: scheduler k (own context, outputs, stream) takes windows k, k+I, ...
    inflight = args.inflight
    if inflight <= 0:  # auto: every scheduler holds its own scratch + packed output
        torch.cuda.synchronize(dev)
        free1 = torch.cuda.mem_get_info(dev)[0]
        per_sched = max(1, free0 - free1)
        inflight = int(min(4, 1 + (0.85 * free1) // per_sched))
    inflight = max(1, inflight)
    scheds = [sched] + [
        WindowScheduler(max_requests=n, max_seq_len=cfg.l_max, n_classes=cfg.n_classes,
                        policies=cfg.policies, split_threshold=cfg.theta, adjust=cfg.adjust,
                        buckets=cfg.init_edges, kv_bytes_per_token=cfg.kvpt,
                        current_safe=cfg.current_safe, accounting=cfg.accounting, device=dev,
                        process_group=pg, dispatch=args.dispatch, pack_capacity=sched.pack_capacity,
                        collective=args.collective)
        for _ in range(inflight - 1)]
    streams = [torch.cuda.Stream(dev) for _ in range(inflight)]

    def run_windows(k_steps, n_inflight):
        cur = torch.cuda.current_stream(dev)
        for st in streams:
            st.wait_stream(cur)
        for i in range(k_steps):
            q = i % n_inflight
            with torch.cuda.stream(streams[q]):
                scheds[q].schedule(lens, cls, tok_off, tokens, sync=False, check=False,
                                   graph=use_graph)
        for st in streams:
            cur.wait_stream(st)

    for q in range(inflight):
        with torch.cuda.stream(streams[q]):
            for _ in range(args.warmup):
                scheds[q].schedule(lens, cls, tok_off, tokens, sync=False, check=False,
                                   graph=use_graph)
    torch.cuda.synchronize(dev)
    # one window at a time (latency per window, reported beside the throughput)
    lat0 = torch.cuda.Event(enable_timing=True)
    lat1 = torch.cuda.Event(enable_timing=True)
    lat_steps = max(3, min(args.steps, 50))
    if pg is not None:
        dist.barrier()
    lat0.record()
    run_windows(lat_steps, 1)
    lat1.record()
    torch.cuda.synchronize(dev)
    window_latency_ms = lat0.elapsed_time(lat1) / lat_steps

    # ---------------- timed region: device-resident windows ----------------------
    sampler = ClockSampler(local_dev)
    l0 = sum(x.ctx.launches for x in scheds)
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    sampler.start()
    time.sleep(0.3)
    # the GPU idled while the sampler started: bring it back to steady state with untimed
    # windows (clocks, caches, the in-flight pipeline's scratch) before the barrier
    run_windows(2 * inflight, inflight)
    if pg is not None:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    run_windows(args.steps, inflight)
    ev1.record()
    torch.cuda.synchronize(dev)
    clocks = sampler.stop()
    if pg is not None:
        dist.barrier()
    launches = sum(x.ctx.launches for x in scheds) - l0
    if use_graph:  # graph replays do not pass through the host launchers: count per window
        launches = kernels_per_window * args.steps
    ms = ev0.elapsed_time(ev1) / args.steps
    for x in scheds:  # check the steady-state result of every scheduler
        s = x.schedule(lens, cls, tok_off, tokens).summary()
        assert s["n_batches"] == s0["n_batches"] and s["packed_elems"] == s0["packed_elems"]
    for x in scheds[1:]:  # release the extra in-flight contexts / outputs before e2e
        x.close()
    del scheds[1:]
    torch.cuda.empty_cache()

    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if pg is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    value = world * n / (ms_max / 1e3)

    # ---------------- pack roofline ------------------------------------------------
    peak, peak_src = _peaks()
    pk_name = _pack_kernel(cfg.l_max, n, cfg.n_classes, args.dispatch, world)
    admitted = int(s["admitted_tokens"])
    n_adm = n - int(s["n_rejected"]) - int(s["n_pending"])
    # SURVEY §8(d) algorithmic bytes: per admitted request 4*len (tokens) + 8 (offset)
    # read; per batch n * max_input_len * (4 + 1) written (int32 token + u8 mask)
    pack_bytes = 4 * admitted + 8 * n_adm + 5 * int(s["padded_tokens"])
    # what K6 actually moves: rows padded to the 16-token pitch, + perm / row map / len
    pack_bytes_pitch = 4 * admitted + 24 * n_adm + 5 * int(s["packed_elems"])
    pack_ms = stage_ms["pack"]
    pack_gbs = pack_bytes / (pack_ms / 1e3) / 1e9 if pack_ms > 0 else None
    sched_bytes = 17 * n
    sched_ms = sum(v for k, v in stage_ms.items() if k != "pack")

    # ---------------- e2e through the public API from pinned host buffers ---------
    e2e = None
    if not args.no_e2e:
        h_lens = lens.cpu().pin_memory()
        h_cls = cls.cpu().pin_memory()
        # the host token store is packed densely (rows 16-byte aligned, the smallest layout
        # the 128-bit pack path accepts) so the PCIe copy moves no padding
        e_off, e_tok = W.token_store_device(lens, seed=rank, align=4)
        h_off = e_off.cpu().pin_memory()
        h_tok = e_tok.cpu().pin_memory()
        del e_off, e_tok
        # two device input sets: the host -> device copies of step i + 1 run on copy streams
        # while step i schedules (the copies dominate: ~33 ms of PCIe per 1M-request window
        # against < 1 ms of GPU work); the token store goes over in 4 slices on 4 streams so
        # both copy engines take part
        dsets = [(torch.empty_like(lens), torch.empty_like(cls), torch.empty_like(h_off, device=dev),
                  torch.empty_like(h_tok, device=dev)) for _ in range(2)]
        nb = int(s["n_batches"])
        h_rb = torch.empty(n, dtype=torch.int32).pin_memory()
        h_bt = torch.empty(64 * nb, dtype=torch.uint8).pin_memory()
        h_sm = torch.empty(256, dtype=torch.uint8).pin_memory()
        copy_streams = [torch.cuda.Stream(dev) for _ in range(4)]
        freed = [torch.cuda.Event() for _ in range(2)]   # compute done with input set k
        for ev in freed:
            ev.record()
        ntok = h_tok.numel()
        n_slices = 4 if ntok * 4 > (256 << 20) else 1  # small windows: one copy stream
        cuts = [ntok * q // n_slices for q in range(n_slices + 1)]

        def e2e_step(i):
            d_l, d_c, d_o, d_t = dsets[i & 1]
            comp = torch.cuda.current_stream(dev)
            landed = []
            for q, cs in enumerate(copy_streams[:n_slices]):
                cs.wait_event(freed[i & 1])
                with torch.cuda.stream(cs):
                    if q == 0:
                        d_l.copy_(h_lens, non_blocking=True)
                        d_c.copy_(h_cls, non_blocking=True)
                        d_o.copy_(h_off, non_blocking=True)
                    d_t[cuts[q]:cuts[q + 1]].copy_(h_tok[cuts[q]:cuts[q + 1]], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    landed.append(ev)
            for ev in landed:
                comp.wait_event(ev)
            # one captured graph per input set (the scheduler keeps both)
            sched.schedule(d_l, d_c, d_o, d_t, sync=False, check=False, graph=use_graph)
            freed[i & 1].record(comp)
            h_rb.copy_(sched.req_batch[:n], non_blocking=True)
            h_bt.copy_(sched.batches_raw[:64 * nb], non_blocking=True)
            h_sm.copy_(sched.summary, non_blocking=True)

        for i in range(2):
            e2e_step(i)
        torch.cuda.synchronize(dev)
        if pg is not None:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        # ~10 steps of a large window (seconds of PCIe), up to 100 of a small one (its
        # ~0.1 ms steps are otherwise at the mercy of host scheduling noise)
        k_e2e = max(3, min(args.steps, 10 if ntok * 4 > (64 << 20) else 100))
        e0.record()
        for cs in copy_streams:  # no copy of the timed steps starts before e0
            cs.wait_stream(torch.cuda.current_stream(dev))
        for i in range(k_e2e):
            e2e_step(i)
        e1.record()
        torch.cuda.synchronize(dev)
        te = torch.tensor([e0.elapsed_time(e1) / k_e2e], dtype=torch.float64, device=dev)
        if pg is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        h2d = h_lens.numel() * 4 + h_cls.numel() + h_off.numel() * 8 + h_tok.numel() * 4
        d2h = n * 4 + 64 * nb + 256
        e2e = {"value": world * n / (float(te.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": float(te.item()), "steps": k_e2e,
               # the copies dominate: the achieved host<->device rate is the e2e roofline
               "pcie_gbs": (h2d + d2h) / (float(te.item()) / 1e3) / 1e9}

    if rank != 0:
        if pg is not None:
            dist.destroy_process_group()
        return

    cpu_base = None
    if not args.no_cpu_baseline and world == 1:
        # the same window as the timed one (capped at 1M requests of host memory)
        if _ALL_CPUS:  # the CPU baseline gets every host core back
            os.sched_setaffinity(0, _ALL_CPUS)
        cpu_base = cpu_baseline(args.config, min(args.cpu_sample or (1 << 20), n))

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        # C5 splits one 64M-request trace over the ranks (total fixed); the others give
        # every rank its own window of the config's size
        "scaling": "strong" if args.config == "c5" else "weak", "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic (seeded lengths per BASELINE config, hashed token ids; generated on device)",
        "impl": "b200",
        "config": {
            "workload": f"{args.config}: {cfg.note}", "requests_per_gpu": n,
            "l_max": cfg.l_max, "classes": cfg.n_classes,
            "kv_bytes_per_token": cfg.kvpt, "safe_memory_bytes": cfg.current_safe,
            "accounting": "padded" if cfg.accounting == 0 else "exact",
            "parallelism": f"dp{world}" if world == 1 else f"dp{world} (request shards, " + {
                "peer": "histogram exchange over CUDA-IPC peer memory inside the window graph)",
                "nccl": "NCCL histogram all-reduce inside the window graph)",
                "torch": f"torch.distributed ({os.environ.get('BS_DIST_BACKEND', 'nccl')}) "
                         "histogram all-reduce between K1 and K2)"}[args.collective],
            "host_binding": (f"{numa_cpus} GPU-local cores (NVML CPU affinity)" if numa_cpus
                             else "unbound"),
            "pipeline": f"{inflight} windows in flight (one scheduler context + CUDA stream each); "
                        "ms_per_step = timed region / steps",
            "l2": "inputs larger than L2 (token store %.2f GB/GPU, packed output %.2f GB/GPU); no flush"
                  % (tokens.numel() * 4 / 1e9, int(s["packed_elems"]) * 5 / 1e9),
        },
        "roofline": {"bound": "hbm", "kernel": pk_name,  # fused windows: K5e wrote the row records
                     "achieved": pack_gbs, "peak": peak,
                     "unit": "GB/s", "frac": (pack_gbs / peak) if pack_gbs else None,
                     "traffic": _profile_traffic(args.config, pk_name), "algorithmic_bytes": pack_bytes,
                     "avg_launch_ms": pack_ms, "peak_source": peak_src,
                     "pitch_overhead": {"bytes_moved": pack_bytes_pitch,
                                        "frac_incl_pitch": (pack_bytes_pitch / (pack_ms / 1e3) / 1e9 / peak)
                                        if pack_ms > 0 else None}},
        "stages_ms": stage_ms,
        "schedule_roofline": {"bytes": sched_bytes, "ms": sched_ms,
                              "achieved_gbs": sched_bytes / (sched_ms / 1e3) / 1e9 if sched_ms else None},
        "window": {"buckets": int(s["k_buckets"]), "n_max": int(s["n_max"]),
                   "batches": int(s["n_batches"]), "rejected": int(s["n_rejected"]),
                   "mean_batch_waste": (s["waste_sum"] / s["n_batches"]) if s["n_batches"] else None},
        "e2e": e2e,
        "cpu_baseline": cpu_base,
        "gpu_launches": launches,
        "cuda_graph": use_graph,
        "inflight": inflight,
        "window_latency_ms": window_latency_ms,
        "c1": None if c1_ms is None else {
            "collective": args.collective, "ms_per_window": c1_ms, "fallback": fallback,
            "bytes": 4 * cfg.l_max * cfg.n_classes,
            "what": "all-reduce (sum) of the uint32 [classes x l_max] length histogram"},
        "clocks": clocks,
    }
    print(json.dumps(line), flush=True)
    if pg is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
