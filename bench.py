#!/usr/bin/env python3
"""bench.py — DPVO front-end fused fake-quant throughput on B200.

Metric (BASELINE.json): "fake-quant GB/s (% of HBM peak) and front-end
frames/sec at 1/2/4/8 B200 vs CPU ref". One STEP = the hot path over one
480x640 frame of BASELINE config 2: per-channel fake-quant forward over the
22 activation quant points of both DPVO encoders (19 tensors, one fused
launch) + the scale-only LSQ/STE backward over the same 22 points (one
launch, bit-exact pairwise-tree scale gradients) [+ at N>1 the NCCL
all-reduce of the 902 per-channel scale gradients, the QAT exchange step].
`value` = frames/s of the whole job; GB/s and the HBM-roofline fraction are
reported beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--dtype f32|f16]
  python bench.py --impl reference ...   # the reference's own CPU code

Under torchrun each rank drives one GPU; frames shard across ranks (weak
scaling, no data-path collective). Timing: CUDA events on the library's
stream, barrier + synchronize on both sides, max over ranks. Inputs are
rotated over >= 2 independent frame sets (> 1.2 GB, >> 126 MB L2).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fake-quant GB/s (% of HBM peak) and front-end frames/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "frames/s"
DATA = "synthetic: standard-normal activations and upstream, per-channel scales log-uniform [1e-3, 0.1]"
WORKLOAD = ("BASELINE config 2: per-channel fake-quant fwd + scale-only LSQ/STE bwd over the 22 "
            "DPVO encoder activation quant points of one 480x640 frame (41,164,800 quant-point elems)")


def parse(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=1000)
    p.add_argument("--warmup", type=int, default=20)
    p.add_argument("--impl", default="qfb", choices=["qfb", "reference"])
    p.add_argument("--dtype", default="f32", choices=["f32", "f16"])
    p.add_argument("--sets", type=int, default=2, help="rotating input sets (L2 defeat)")
    p.add_argument("--e2e-steps", type=int, default=60)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                   help="gloo: exercise the N>1 path with ranks sharing one GPU (tests only)")
    p.add_argument("--graph-steps", type=int, default=8,
                   help="consecutive steps captured in one CUDA graph (N=1)")
    p.add_argument("--no-single-thread", action="store_true",
                   help="reference arm: skip the one-thread sample")
    p.add_argument("--no-secondary", action="store_true",
                   help="skip the config-3 chain window and config-5 forward-throughput lines")
    p.add_argument("--async-finish", action="store_true",
                   help="run the backward's finisher on the library's side stream (QFB_OPT_BWD_ASYNC_FINISH, "
                        "joined by the next step's backward / the end of the timed region); measured slower "
                        "for f32 (the finisher's CTAs delay the persistent forward's first wave)")
    p.add_argument("--half-fp32-terms", action="store_true",
                   help="f16: the opt-in float32-term backward (QFB_OPT_BWD_HALF_FP32; d_input bitwise, "
                        "scale gradients within tolerance instead of bitwise)")
    return p.parse_args(argv)


def parse_args_list(argv):
    return parse(argv)


# ------------------------------------------------------------- helpers --

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def load_traffic():
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu
    capture summary (profiles/ncu_traffic.json), else None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------ reference (CPU) --

class RefCpuWorkload:
    """The reference's own per-channel fake_quantize (quant.hpp:150) and
    fake_quantize_backward (quant.hpp:261), compiled -O3 from its sources
    (oracle/_ref), over the frame's 22 quant points. Work items are
    4-channel blocks (the per-channel ops are independent per channel, so
    blocking does not change the work), pulled by `threads` host threads.
    A bounded sample (a fixed subset of blocks, sized to `budget_s`) is
    timed and converted to frames/s = frames-worth of elements / seconds."""

    def __init__(self, consumers, threads, dtype="f32", seed=7, do_bwd=True, mode="blocks", lib=None):
        import numpy as np
        import oracle
        self.ref = oracle.Reference(lib) if lib else oracle.Reference()
        self.lib = os.path.basename(lib) if lib else "libqfref.so"
        self.mode = mode  # "blocks": 4-channel blocks over a pool; "sweeps": the reference's schedule
        self.threads = threads
        self.do_bwd = 1 if do_bwd else 0
        self.reps = 1
        self.half = 1 if dtype == "f16" else 0
        rng = np.random.default_rng(seed)
        self.items = []
        self.frame_elems = sum(p.numel for (p, _c) in consumers)
        xs = {}
        for (p, _c) in consumers:
            if p.name not in xs:
                xs[p.name] = rng.standard_normal((p.channels, p.inner), dtype=np.float32)
            x = xs[p.name]
            up = rng.standard_normal((p.channels, p.inner), dtype=np.float32)
            ls = np.log(np.expm1(np.exp(rng.uniform(np.log(1e-3), np.log(0.1), p.channels))))
            step = 4 if mode == "blocks" else p.channels
            for c0 in range(0, p.channels, step):
                c1 = min(c0 + step, p.channels)
                self.items.append((np.ascontiguousarray(x[c0:c1]), np.ascontiguousarray(up[c0:c1]),
                                   c1 - c0, p.inner, np.ascontiguousarray(ls[c0:c1])))
        order = list(range(len(self.items)))
        rng.shuffle(order)
        self.order = order
        self.sel = order

    def _run(self, idx, reps=1):
        sel = [self.items[i] for i in idx]
        if self.mode == "sweeps":
            st, secs, _ = self.ref.bench_sweeps([s[0] for s in sel], [s[1] for s in sel],
                                                [s[2] for s in sel], [s[3] for s in sel],
                                                [s[4] for s in sel], half=self.half,
                                                do_bwd=self.do_bwd, threads=self.threads, reps=reps)
        else:
            st, secs, _ = self.ref.bench_points([s[0] for s in sel], [s[1] for s in sel],
                                                [s[2] for s in sel], [s[3] for s in sel],
                                                [s[4] for s in sel], half=self.half,
                                                do_bwd=self.do_bwd, threads=self.threads, reps=reps)
        assert st == 0, f"reference bench failed: {st}"
        return secs, reps * sum(s[2] * s[3] for s in sel)

    def size(self, budget_s):
        """Pick the sample: a subset of one frame's blocks when a frame takes
        longer than the budget, else whole frames repeated (reps) to fill it."""
        probe = self.order[:max(2 * self.threads, 8)] if self.mode == "blocks" else self.order[:2]
        secs, elems = self._run(probe)
        want = elems / max(secs, 1e-9) * budget_s
        self.reps = 1
        if want >= self.frame_elems:
            self.sel = self.order
            secs, elems = self._run(self.sel)          # one full frame, warm
            self.reps = max(1, int(round(budget_s / max(secs, 1e-9))))
            return self
        acc, k = 0, 0
        while k < len(self.order) and acc < want:
            it = self.items[self.order[k]]
            acc += it[2] * it[3]
            k += 1
        self.sel = self.order[:max(k, min(len(self.order), self.threads))]
        return self

    def run(self):
        secs, elems = self._run(self.sel, self.reps)
        return secs, elems / self.frame_elems

    def describe(self, secs, frames):
        if self.mode == "sweeps":
            return (f"{frames:.3f} frames-worth of quant-point elements ({len(self.sel)} of "
                    f"{len(self.items)} quant points x {self.reps} reps) in {secs:.2f} s; the reference's own "
                    f"schedule: scale pass + fused sweep through qf::Dispatcher({self.threads}) (exec.hpp:127-146, "
                    f"248-259, 363-375) + sequential fake_quantize_backward (frontend.hpp:226-229); {self.lib}")
        ops = "fake_quantize + fake_quantize_backward" if self.do_bwd else "fake_quantize"
        return (f"{frames:.3f} frames-worth of quant-point elements ({len(self.sel)} of "
                f"{len(self.items)} 4-channel blocks x {self.reps} reps) in {secs:.2f} s on "
                f"{self.threads} threads; reference quant.hpp {ops}, -O3 from its sources ({self.lib})")


def reference_variants(consumers, threads, dtype, budget_s=3.0):
    """The other CPU lines BASELINE.md §3 names, each a bounded sample:
    the reference's own schedule (ExecutionPlan.threads = all host threads
    and 0) and the channel-block pool built for x86-64-v3 (the -march=native
    line; FMA contraction may change bits, timing only)."""
    import oracle
    out = {}
    for key, th in (("reference_schedule_threads_all", threads), ("reference_schedule_threads_0", 0)):
        w = RefCpuWorkload(consumers, th, dtype, mode="sweeps").size(budget_s)
        s_, f_ = w.run()
        out[key] = {"value": f_ / s_, "unit": UNIT, "cores": max(th, 1), "sample": w.describe(s_, f_)}
    if os.path.exists(oracle.REF_V3_PATH):
        try:
            w = RefCpuWorkload(consumers, threads, dtype, lib=oracle.REF_V3_PATH).size(budget_s)
            s_, f_ = w.run()
            out["march_x86_64_v3"] = {"value": f_ / s_, "unit": UNIT, "cores": threads,
                                      "sample": w.describe(s_, f_)}
        except OSError as e:  # a host CPU without AVX2/FMA
            out["march_x86_64_v3"] = {"unavailable": str(e)}
    return out


def cpu_reference_frames_per_s(consumers, budget_s, threads, dtype="f32", do_bwd=True):
    import oracle
    if not oracle.reference_available():
        return None
    w = RefCpuWorkload(consumers, threads, dtype, do_bwd=do_bwd).size(budget_s)
    secs, frames = w.run()
    out = {"value": frames / secs, "unit": UNIT, "cores": threads, "kind": "reference",
           "sample": w.describe(secs, frames), "host": host_cpu_info()}
    if threads > 1:
        # the reference at threads = 0 (sequential) as well
        w1 = RefCpuWorkload(consumers, 1, dtype, do_bwd=do_bwd).size(min(5.0, budget_s / 3))
        s1, f1 = w1.run()
        out["single_thread"] = {"value": f1 / s1, "unit": UNIT, "cores": 1, "sample": w1.describe(s1, f1)}
    return out


def host_cpu_info():
    """hardware_concurrency, the affinity mask and the cgroup CPU quota."""
    info = {"hardware_concurrency": os.cpu_count(), "affinity": host_threads()}
    try:
        q = open("/sys/fs/cgroup/cpu.max").read().split()
        info["cgroup_cpu_max"] = None if q[0] == "max" else int(q[0]) / int(q[1])
    except Exception:
        info["cgroup_cpu_max"] = None
    return info


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def bench_config(args, ws):
    """The `config` object of the JSON line — one function for both arms,
    so the reference arm and ours describe the identical workload (same
    dict, byte for byte)."""
    from paper_2511_12653_b200.shapes import dpvo_quant_points, frame_bytes
    pts = dpvo_quant_points()
    esize = 4 if args.dtype == "f32" else 2
    b = frame_bytes(pts, esize)
    step_bytes = b["fwd"] + b["bwd"]
    return {"workload": WORKLOAD, "frames_per_step_per_gpu": 1,
            "quant_points": sum(len(p.consumers) for p in pts), "tensors": len(pts),
            "scales": "per-channel, log-uniform [1e-3, 0.1]",
            "l2_policy": f"inputs > L2: {max(1, args.sets)} rotating frame sets, "
                         f"{step_bytes / 1e6:.0f} MB moved per step vs 126 MB L2",
            "parallelism": (f"frames sharded over {ws} GPUs (one process each); per step one "
                            f"exchange of the per-frame scale-gradient rows: NCCL all-gather + "
                            f"frame-order fold through the C-ABI (qfb_gather_fold_scale_grads)"
                            if ws > 1 else "1 GPU"),
            **({"backward_terms": "float32 (QFB_OPT_BWD_HALF_FP32): d_input bitwise, scale gradients "
                                  "within the FP16 tolerance, not bitwise"}
               if getattr(args, "half_fp32_terms", False) else {})}


def run_reference_arm(args):
    """--impl reference: the reference CPU implementation on the host cores,
    same metric/unit/config; each step a bounded sample of the workload.
    This process maps no native code of the package (shapes is pure
    Python); the timed code is the reference's, compiled from its sources
    (oracle/_ref/libqfref.so)."""
    import oracle
    from paper_2511_12653_b200.shapes import dpvo_quant_points
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    if not oracle.reference_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libqfref.so missing"}))
        return 0
    pts = dpvo_quant_points()
    consumers = [(p, c) for p in pts for c in p.consumers]
    threads = host_threads()
    per_step = max(0.02, min(2.0, 120.0 / max(1, args.steps + args.warmup)))
    w = RefCpuWorkload(consumers, threads, args.dtype).size(per_step)
    for _ in range(args.warmup):
        w.run()
    tot_s, tot_f = 0.0, 0.0
    for _ in range(args.steps):
        s, f = w.run()
        tot_s += s
        tot_f += f
    fps = tot_f / tot_s
    cpu = {"value": fps, "unit": UNIT, "cores": threads, "kind": "reference",
           "sample": "per step: " + w.describe(tot_s / args.steps, tot_f / args.steps),
           "host": host_cpu_info()}
    if not args.no_single_thread:
        # the reference at threads = 0 (sequential) as well
        w1 = RefCpuWorkload(consumers, 1, args.dtype).size(3.0)
        s1, f1 = w1.run()
        cpu["single_thread"] = {"value": f1 / s1, "unit": UNIT, "cores": 1, "sample": w1.describe(s1, f1)}
        cpu.update(reference_variants(consumers, threads, args.dtype))
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 / fps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": DATA,
            "data_generator": "numpy default_rng standard normal on the host",
            "config": bench_config(args, ws),
            "impl": "reference",
            "cpu_baseline": cpu,
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def reference_arm_subprocess(args, steps=8, warmup=2):
    """cpu_baseline of our arm: the reference arm itself (`bench.py --impl
    reference`), run as a fresh process with the same dtype, so the two
    numbers are the same code under the same conditions."""
    env = {k: v for k, v in os.environ.items()
           if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    cmd = [sys.executable, os.path.abspath(__file__), "--impl", "reference", "--steps", str(steps),
           "--warmup", str(warmup), "--dtype", args.dtype, "--sets", str(args.sets)]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=600)
    for ln in out.stdout.splitlines()[::-1]:
        ln = ln.strip()
        if ln.startswith("{"):
            d = json.loads(ln)
            if "unavailable" in d:
                return None
            cpu = dict(d["cpu_baseline"])
            cpu["sample"] = (f"`bench.py --impl reference --steps {steps} --warmup {warmup}` in a fresh "
                             f"process: " + cpu["sample"])
            return cpu
    raise RuntimeError(f"reference arm failed: rc={out.returncode} {out.stderr[-400:]}")


# --------------------------------------------------------- our arm (GPU) --

class Plumbing:
    """N > 1 process plumbing. torch.distributed runs on gloo for control
    only (the NCCL id broadcast, barriers, the max over ranks of the timed
    region); the data exchange of the QAT step — the per-frame scale-gradient
    rows, all-gathered and folded in global frame order — goes through the
    library's C-ABI on NCCL (qfb_nccl_comm_init_rank +
    qfb_gather_fold_scale_grads, captured in the step's CUDA graph).
    --dist-backend gloo (tests: ranks sharing one GPU, where NCCL refuses
    to run) exchanges the rows through gloo instead, eagerly."""

    def __init__(self, args, q, ws, rank, gpu):
        import torch.distributed as dist
        self.ws, self.rank, self.gpu, self.dist = ws, rank, gpu, dist
        self.nccl = args.dist_backend == "nccl"
        dist.init_process_group("gloo")
        self.comm = None
        if self.nccl:
            box = [q.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(box, src=0)
            self.comm = q.NcclRankComm(box[0], ws, rank, gpu)

    def exchange(self, ctx, rows_per_rank, n, device):
        from paper_2511_12653_b200.frontend import GlooGatherFold, NcclGatherFold
        if self.nccl:
            return NcclGatherFold(ctx, self.comm, rows_per_rank, n, device=device)
        return GlooGatherFold(ctx)

    def barrier(self):
        self.dist.barrier()

    def max(self, v: float) -> float:
        import torch
        t = torch.tensor([float(v)], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.comm is not None:
            self.comm.close()
        self.dist.barrier()
        self.dist.destroy_process_group()


def run_qfb(args):
    import torch

    import paper_2511_12653_b200 as q
    from paper_2511_12653_b200.frontend import FrontendQuantPass

    ws, rank, local = dist_env()
    # --dist-backend gloo (test only): ranks may share a GPU, so the device is
    # local % device_count; with NCCL (the default) every rank owns a GPU
    gpu = local % max(1, torch.cuda.device_count()) if args.dist_backend == "gloo" else local
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    pg = Plumbing(args, q, ws, rank, gpu) if ws > 1 else None
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    ctx = q.Context(gpu, stream.cuda_stream)
    if args.half_fp32_terms:
        ctx.set_option(q.OPT_BWD_HALF_FP32, 1)
    # at N > 1 the step's backward leaves this rank's frame row for the
    # exchange; every rank holds distinct frames (frame_offset = rank)
    rows = None
    if ws > 1:
        from paper_2511_12653_b200.shapes import dpvo_quant_points
        n_grad = sum(p.channels * len(p.consumers) for p in dpvo_quant_points())
        rows = torch.zeros((1, n_grad), dtype=torch.float64, device=dev)
    fp = FrontendQuantPass(ctx, frames=1, dtype=args.dtype, sets=max(1, args.sets), seed=1, device=dev,
                           rows_out=rows, frame_offset=rank)
    grads = fp.scale_grads()
    nsets = len(fp.sets)
    ex = pg.exchange(ctx, 1, fp.n_grad, dev) if pg is not None else None

    def exchange():
        if ex is not None:
            # QAT exchange: the step's frame rows of all ranks, folded in
            # frame order into the gradient vector (bit-identical at any N)
            ctx.join()  # the rows are complete once the finisher is joined
            ex(rows, grads)

    def eager_step(i, ev=None):
        si = i % nsets
        if ev is not None:
            ev[0].record(stream)
            # the library records ev[3] between the backward's main pass and
            # its finisher (QFB_OPT_MAIN_PASS_EVENT): the dominant kernel alone
            ctx.set_option(q.OPT_MAIN_PASS_EVENT, ev[3].cuda_event)
        fp.forward(si)
        if ev is not None:
            ev[1].record(stream)
        fp.backward(si)
        if ev is not None:
            ctx.join()  # the finisher inside the measured backward
            ev[2].record(stream)
            ctx.set_option(q.OPT_MAIN_PASS_EVENT, 0)
        exchange()

    # warm up eagerly (sizes the workspaces), then capture the step as CUDA
    # graphs: 1 forward + 2 backward launches (+ the NCCL exchange at N > 1)
    for i in range(max(1, args.warmup)):
        eager_step(i)
    ctx.sync()
    # the finisher of step k overlaps the forward of step k+1 (side stream,
    # joined by step k+1's backward and at the end of every captured graph)
    if args.async_finish:
        ctx.set_option(q.OPT_BWD_ASYNC_FINISH, 1)
    capturable = pg is None or pg.nccl
    use_graph = not args.no_graph and capturable
    graphs = []
    launches_per_step = 3
    # steps per graph replay: G consecutive steps (sets alternating) in one
    # graph, so the per-replay launch gap is paid once per G steps
    G = max(1, args.graph_steps)
    G = G - G % nsets if G >= nsets else G
    big = None
    if use_graph:
        try:
            c0 = ctx.launch_count
            for si in range(nsets):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    fp.forward(si)
                    fp.backward(si)
                    exchange()
                    ctx.join()
                graphs.append(g)
            launches_per_step = (ctx.launch_count - c0) // nsets
            if G > 1:
                big = torch.cuda.CUDAGraph()
                with torch.cuda.graph(big, stream=stream):
                    for k in range(G):
                        fp.forward(k % nsets)
                        fp.backward(k % nsets)
                        exchange()
                    ctx.join()
        except Exception as exc:  # pragma: no cover - fall back to eager timing
            print(f"graph capture failed ({exc}); timing eager launches", file=sys.stderr)
            use_graph = False
            big = None
    elif pg is not None:
        c0 = ctx.launch_count
        eager_step(0)
        launches_per_step = ctx.launch_count - c0

    def step(i):
        if use_graph:
            graphs[i % nsets].replay()
        else:
            eager_step(i)

    def run_steps(k):
        """k consecutive steps from step 0 (set order preserved)."""
        i = 0
        if big is not None:
            for _ in range(k // G):
                big.replay()
            i = (k // G) * G
        while i < k:
            step(i)
            i += 1

    for i in range(args.warmup):
        step(i)
    if big is not None:
        big.replay()
    ctx.sync()
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize(dev)

    sampler = ClockSampler(gpu)
    sampler.start()
    time.sleep(0.15)  # let the sampler attach before the timed region
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    wall0 = time.perf_counter()
    t_start.record(stream)
    run_steps(args.steps)
    ctx.join()  # eager path: the last step's finisher
    t_end.record(stream)
    torch.cuda.synchronize(dev)
    wall1 = time.perf_counter()
    clocks = sampler.stop()
    launches = launches_per_step * args.steps
    ctx.sync()
    ms_total = t_start.elapsed_time(t_end)

    # per-kernel attribution for the roofline: the same steps launched
    # eagerly with CUDA events around each kernel on the library's stream
    k_att = min(args.steps, 200)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(k_att)]
    for e in evs:
        e[3].record(stream)  # creates the CUDA event the library records into
    torch.cuda.synchronize(dev)
    for i in range(k_att):
        eager_step(i, evs[i])
    torch.cuda.synchronize(dev)
    ctx.set_option(q.OPT_BWD_ASYNC_FINISH, 0)  # stream-ordered finisher for everything below
    fwd_ms = sum(e[0].elapsed_time(e[1]) for e in evs) / k_att
    bwd_ms = sum(e[1].elapsed_time(e[2]) for e in evs) / k_att
    bwd_main_ms = sum(e[1].elapsed_time(e[3]) for e in evs) / k_att
    fin_ms = sum(e[3].elapsed_time(e[2]) for e in evs) / k_att
    if pg is not None:
        ms_total = pg.max(ms_total)
        pg.barrier()
    ms_step = ms_total / args.steps
    frames_total = ws * args.steps * fp.frames
    fps = frames_total / (ms_total / 1000.0)
    b = fp.bytes_per_step()
    step_bytes = b["fwd"] + b["bwd"]
    gbps = ws * step_bytes / (ms_step / 1000.0) / 1e9
    peak, peak_src = load_peaks()
    fwd_gbps = b["fwd"] / (fwd_ms / 1000.0) / 1e9
    bwd_gbps = b["bwd"] / (bwd_ms / 1000.0) / 1e9
    traffic = load_traffic()
    dominant = "bwd" if b["bwd"] >= b["fwd"] else "fwd"
    bwd_main_gbps = b["bwd"] / (bwd_main_ms / 1000.0) / 1e9
    roofline = {"bound": "hbm", "kernel": "qfb::bwd_kernel (scale-only LSQ/STE backward, main pass)",
                "achieved": bwd_main_gbps, "peak": peak, "unit": "GB/s", "frac": bwd_main_gbps / peak,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": b["bwd"],
                "launch_us": bwd_main_ms * 1e3,
                "with_finisher": {"kernels": "bwd_kernel + bwd_finish_reg_kernel (one C-ABI call)",
                                  "us": bwd_ms * 1e3, "achieved": bwd_gbps, "frac": bwd_gbps / peak,
                                  "finisher_us": fin_ms * 1e3},
                "timing": "CUDA events on the library stream around each kernel of 200 eager steps inside "
                          "the bench (the library records the main-pass event between its two launches, "
                          "QFB_OPT_MAIN_PASS_EVENT); algorithmic bytes = 3 x 4 B x 41,164,800 quant-point "
                          "elements (read x and upstream, write d_input)",
                "traffic": (traffic or {}).get(args.dtype, {}).get("bwd_bytes_per_launch"),
                "fwd_kernel": {"kernel": "qfb::ew_tma_kernel<T, false, NS> (fused multi-point forward; "
                                         "NS = tma_stages(): 3 for one f32 frame)",
                               "achieved": fwd_gbps, "frac": fwd_gbps / peak,
                               "algorithmic_bytes_per_launch": b["fwd"],
                               "traffic": (traffic or {}).get(args.dtype, {}).get("fwd_bytes_per_launch")},
                "step_gbps": gbps / ws, "step_frac": (gbps / ws) / peak}

    # ---------------------------------------------------- e2e (host API) --
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, q, ctx, fp, stream, dev, pg, ws, rank)

    secondary = None
    if not args.no_secondary:
        secondary = run_secondary(args, ctx, stream, dev, peak, rank, ws, pg)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            cpu = reference_arm_subprocess(args)
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": UNIT, "cores": host_threads(), "kind": "reference",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
                "data": DATA,
                "data_generator": "CounterRng normal (rng.hpp:24-50), generated on the device",
                "config": bench_config(args, ws),
                "gbps": gbps, "hbm_frac": (gbps / ws) / peak,
                "kernel_ms": {"fwd": fwd_ms, "bwd": bwd_ms, "bwd_main": bwd_main_ms, "bwd_finish": fin_ms},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "secondary": secondary,
                "finisher": ("stream-ordered" if not args.async_finish else
                             "side stream (QFB_OPT_BWD_ASYNC_FINISH): step k's finisher overlaps step k+1's "
                             "forward, joined by step k+1's backward and before the end of the timed region"),
                "timing": (f"value: CUDA-graph replays of {G} consecutive steps each (fwd + bwd + finisher "
                           "launches per step" + (" + the NCCL gather-fold exchange" if ws > 1 else "") +
                           ", serial on the library stream) between CUDA events, max over ranks"
                           if use_graph else
                           "value: eager launches between CUDA events on the library stream") +
                          f"; roofline: per-kernel CUDA events over {k_att} eager steps",
                "wall_ms_per_step": (wall1 - wall0) * 1000.0 / args.steps}
        print(json.dumps(line))
    ctx.close()
    if pg is not None:
        pg.close()
    return 0


def time_device(fn, stream, reps, warmup=2):
    """ms per call of fn() on `stream` (CUDA events, synchronized)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(reps):
        fn()
    t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / reps


def time_aggregate(fn, n_calls, stream, pg, warmup=2):
    """ms for n_calls calls of fn() on this rank (CUDA events on `stream`),
    the whole job's time = the max over ranks, barrier + synchronize on both
    sides."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if pg is not None:
        pg.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(n_calls):
        fn()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    if pg is not None:
        ms = pg.max(ms)
        pg.barrier()
    return ms


def run_secondary(args, ctx, stream, dev, peak, rank, ws, pg):
    """BASELINE configs 3, 5, 4 and 1 on this GPU (reported beside the
    headline): c3 = fused quant->act->quant chains over every quant point of
    a 15-frame window + its patch/update-operator inputs (ReLU and GELU);
    c5 = the throughput sweep as specified: 32 sequences x 1000 frames
    through the fused forward, sequences split over the ranks, 8 frames per
    launch, timed as one aggregate (max over ranks); c4 = the 64-frame QAT
    step; c1 = the per-tensor map."""
    import torch
    from paper_2511_12653_b200.frontend import FrontendQuantPass, WindowChainPass
    out = {}
    for gelu in (False, True):
        wp = WindowChainPass(ctx, frames=15, patches=96, gelu=gelu, dtype=args.dtype, device=dev)
        ms = time_device(wp.run, stream, reps=10)
        gb = wp.bytes_per_run() / (ms / 1e3) / 1e9
        out["c3_chain_window_" + ("gelu" if gelu else "relu")] = {
            "ms_per_window": ms, "gbps": gb, "hbm_frac": gb / peak,
            "bytes_per_window": wp.bytes_per_run(), "quant_points": len(wp.points),
            "launches_per_window": 1,
            "workload": "15-frame window: 22 encoder quant points x 15 frames + gmap/imap (96 patches x "
                        "15) + corr/net/inp (21,600 edges), relu(a [+ b]) or gelu -> K fake-quant outputs" +
                        ("; GELU is defined by this build (the reference has none: parity unpinned, "
                         "oracle and kernel share include/qfb_portable.h)" if gelu else "")}
        del wp
        torch.cuda.empty_cache()
    for int8 in (False, True):
        fp = FrontendQuantPass(ctx, frames=8, dtype=args.dtype, sets=2, seed=11, device=dev, int8_out=int8,
                               frame_offset=8 * rank)
        k = [0]

        def fwd():
            fp.forward(k[0] % 2)
            k[0] += 1
        total = 32 * 1000
        per_rank = total // ws
        launches = (per_rank + fp.frames - 1) // fp.frames
        ms = time_aggregate(fwd, launches, stream, pg)
        fps = ws * launches * fp.frames / (ms / 1e3)
        key = "fwd_int8" if int8 else "fwd"
        gb = ws * launches * fp.bytes_per_step()[key] / (ms / 1e3) / 1e9
        line = {"value": fps, "unit": "frames/s", "seconds_for_32x1000_frames": ms / 1e3,
                "gbps_per_gpu": gb / ws, "hbm_frac": gb / ws / peak, "frames_per_launch": fp.frames,
                "launches_per_rank": launches, "n_gpus": ws,
                "timing": "all 32,000 frames (32 sequences x 1000) split over the ranks; CUDA events around "
                          "each rank's launches, barrier + synchronize both sides, max over ranks"}
        if int8:
            line["workload"] = ("config 5 forward emitting int8 codes (QFB_FLAG_INT8_OUT, SURVEY §8 f2): "
                                "input read once, 1 byte written per quant-point element")
            out["c5_forward_int8_codes"] = line
        else:
            line["workload"] = ("BASELINE config 5: fused multi-point fake-quant forward of the 22 DPVO "
                                "activation quant points (inference front-end) over 32 x 1000 frames, 8 frames "
                                "per launch; weights are fake-quantized once (cache_weights, exec.hpp:59-60)")
            if rank == 0 and ws == 1 and not args.no_cpu:
                cons = [(p, c) for p in fp.points for c in p.consumers]
                try:
                    line["cpu_baseline"] = cpu_reference_frames_per_s(cons, 5.0, host_threads(), args.dtype,
                                                                      do_bwd=False)
                except Exception as exc:  # pragma: no cover
                    line["cpu_baseline"] = {"value": None, "sample": f"failed: {exc}"}
            out["c5_forward_throughput"] = line
        del fp
        torch.cuda.empty_cache()
    out["c4_qat_step"] = run_qat_step(args, ctx, stream, dev, peak, rank, ws, pg)
    out["c1_per_tensor_fwd"] = run_c1(args, ctx, stream, dev, peak, rank, ws)
    return out


def run_c1(args, ctx, stream, dev, peak, rank, ws):
    """BASELINE config 1: per-tensor fake-quant forward of the fnet output
    map [1, 128, 120, 160]: the latency of one call (inputs
    resident) and GB/s over 128 rotating distinct maps (2.5 GB >> L2); the
    reference's fake_quantize on one host thread beside it."""
    import torch
    import paper_2511_12653_b200 as q
    n = 128 * 120 * 160
    tdt = torch.float32 if args.dtype == "f32" else torch.float16
    esize = 4 if args.dtype == "f32" else 2
    L = q.lib()
    xs = torch.empty((128, n), dtype=tdt, device=dev)
    q.check(L.qfb_fill_rng(ctx.handle, 0 if args.dtype == "f32" else 1, xs.data_ptr(), xs.numel(), 1, 0, 0, 1,
                           1.0, 0.0))
    ys = torch.empty_like(xs)
    s = torch.tensor([q.resolve_scale([q.softplus_inv(4.0 / 127)])[0]], dtype=torch.float32, device=dev)
    dt = 0 if args.dtype == "f32" else 1
    k = [0]

    def one():
        i = k[0] % 128
        k[0] += 1
        q.check(L.qfb_fq_fwd(ctx.handle, dt, xs[i].data_ptr(), ys[i].data_ptr(), 1, 1, n, s.data_ptr(), 127, 0))
    lat = time_device(one, stream, reps=1, warmup=3)
    ms_eager = time_device(one, stream, reps=256, warmup=8)
    # the same 128 calls captured once as a CUDA graph: device time per call
    # without the Python/ctypes launch cost of the eager loop
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(128):
            one()
    ms = time_device(g.replay, stream, reps=4, warmup=2) / 128
    # one call as a one-node graph: its device latency without the host launch path
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=stream):
        one()
    lat_dev = time_device(g1.replay, stream, reps=1, warmup=3)
    gb = 2 * n * esize / (ms / 1e3) / 1e9
    res = {"us_single_call": lat * 1e3, "us_single_call_device": lat_dev * 1e3,
           "us_per_call_rotating_eager": ms_eager * 1e3,
           "us_per_call_rotating": ms * 1e3, "gbps": gb, "hbm_frac": gb / peak,
           "workload": "BASELINE config 1: per-tensor fake-quant fwd of [1,128,120,160], 128 rotating maps",
           "timing": "us_single_call: one eager call after warm-up (host launch path included); "
                     "us_single_call_device: the same call replayed as a one-node graph; "
                     "us_per_call_rotating / gbps: 128 calls "
                     "over distinct maps (2.5 GB) replayed as one CUDA graph; _eager: the same calls "
                     "launched one by one from Python"}
    if rank == 0 and ws == 1 and not args.no_cpu:
        try:
            import numpy as np
            import oracle
            if oracle.reference_available():
                ref = oracle.Reference()
                x = xs[0].float().cpu().numpy().reshape(1, 128, 120, 160)
                sv = float(s.item())
                ref.fake_quantize(x, x.shape, [sv])            # warm
                t0 = time.perf_counter()
                reps = 5
                for _ in range(reps):
                    ref.fake_quantize(x, x.shape, [sv])
                cpu_ms = (time.perf_counter() - t0) * 1e3 / reps
                res["cpu_baseline"] = {"ms_per_call": cpu_ms, "cores": 1, "kind": "reference",
                                       "sample": f"{reps} calls of qf::fake_quantize per-tensor on the "
                                                 f"same map, one host thread"}
        except Exception as exc:  # pragma: no cover
            res["cpu_baseline"] = {"value": None, "sample": f"failed: {exc}"}
    del xs, ys, g, g1
    torch.cuda.empty_cache()
    return res


def run_qat_step(args, ctx, stream, dev, peak, rank, ws, pg):
    """BASELINE config 4: one scale-only QAT step over 64 frames, sharded
    64 / N per rank: fused fake-quant forward, per-frame distillation loss
    (fnet and inet pairs), scale-only backward leaving one gradient row per
    frame, the rows of all ranks gathered and folded in frame order (NCCL
    through the C-ABI at N > 1), then Adam (device step counter) — replicas
    stay bitwise equal. Scales are resolved on the device from the current
    log scales each step. Convolutions excluded (cuDNN); features and
    upstream are synthetic. The step replays as one CUDA graph."""
    import torch
    from paper_2511_12653_b200.frontend import QatStep
    frames = max(1, 64 // ws)
    qs = QatStep(ctx, frames=frames, dtype=args.dtype, seed=21, device=dev, frame_offset=rank * frames,
                 total_frames=frames * ws, resolve="device")
    if pg is not None:
        qs.exchange_fn = pg.exchange(ctx, frames, qs.n_act, dev)
    qs.run()  # sizes the scratch (growth is refused under capture)
    torch.cuda.synchronize(dev)
    runner = qs.run
    graph = pg is None or pg.nccl
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            qs.run()
        runner = g.replay
    ms = time_aggregate(runner, 5, stream, pg, warmup=1)
    gb = qs.bytes_per_step() / (ms / 5 / 1e3) / 1e9
    res = {"ms_per_step": ms / 5, "frames_per_step": frames * ws, "frames_per_s": frames * ws / (ms / 5 / 1e3),
           "gbps_per_gpu": gb, "hbm_frac": gb / peak, "n_gpus": ws,
           "scaling": "strong (64 frames over N GPUs)", "graph": graph,
           "workload": "BASELINE config 4: scale-only QAT step over 64 frames (device scale resolve, fwd FQ "
                       "22 points, distill loss fnet+inet per frame, bwd FQ with per-frame rows, frame-order "
                       "gather-fold of the rows over all ranks, Adam on 1,494 scales); convolutions excluded"}
    del qs
    if graph:
        del g
    torch.cuda.empty_cache()
    return res


def run_e2e(args, q, ctx, fp, stream, dev, pg, ws, rank):
    """Same workload end to end through the public host C-ABI: one
    qfb_quant_pass_host_submit / _wait pair per frame (pinned host float32
    buffers in: every quant-point tensor + every upstream; host buffers out:
    every FQ output, d_input and scale gradient). Two frames are in flight
    (two host buffer sets, slots 0/1), so frame k+1's uploads run under frame
    k's downloads; every frame's copies are inside the timed region."""
    import ctypes

    import numpy as np
    import torch
    L = q.lib()
    cfg = q.QuantConfig().to_c()
    keep = []

    def build(set_index):
        # the frame's host buffers: one pinned input arena (per point: x,
        # then its consumers' upstreams) and one pinned output arena (per
        # point and consumer: y, then d_input) — the library's copy order,
        # so its contiguous copies merge (fewer DMA operations per frame)
        r16 = lambda n: (n + 3) & ~3  # noqa: E731  (16-byte aligned float offsets)
        n_in = sum(r16(p.numel) * (1 + len(p.consumers)) for p in fp.points)
        n_out = sum(2 * r16(p.numel) * len(p.consumers) for p in fp.points)
        a_in = torch.empty(n_in, dtype=torch.float32).pin_memory()
        a_out = torch.empty(n_out, dtype=torch.float32).pin_memory()
        keep.extend([a_in, a_out])
        o_in, o_out = [0], [0]

        def take(arena, off, n):
            t = arena[off[0]:off[0] + n]
            off[0] += r16(n)
            return t

        pts, grad_arrays = [], []
        ci = 0
        for pi, p in enumerate(fp.points):
            hx = take(a_in, o_in, p.numel)
            hx.copy_(fp.sets[set_index % len(fp.sets)]["x"][pi].reshape(-1).float().cpu())
            hp = q.CHostPoint()
            hp.x = hx.data_ptr()
            hp.outer, hp.channels, hp.inner, hp.n_out = 1, p.channels, p.inner, len(p.consumers)
            for k in range(len(p.consumers)):
                ls = np.ascontiguousarray(fp.log_s[ci], dtype=np.float64)
                sc = np.array(q.resolve_scale(ls.tolist()), dtype=np.float64)
                hup = take(a_in, o_in, p.numel)
                hup.copy_(fp.sets[set_index % len(fp.sets)]["up"][ci].reshape(-1).float().cpu())
                hy = take(a_out, o_out, p.numel)
                hdx = take(a_out, o_out, p.numel)
                dls = np.zeros(p.channels, dtype=np.float64)
                keep.extend([ls, sc, dls])
                grad_arrays.append(dls)
                hp.s[k], hp.y[k], hp.log_s[k] = sc.ctypes.data, hy.data_ptr(), ls.ctypes.data
                hp.up[k], hp.dx[k], hp.d_log_s[k] = hup.data_ptr(), hdx.data_ptr(), dls.ctypes.data
                ci += 1
            pts.append(hp)
        return (q.CHostPoint * len(pts))(*pts), len(pts), grad_arrays

    tables = [build(0), build(1)]
    prec = 1 if args.dtype == "f16" else 0

    n_grad = sum(p.channels for (p, _c) in fp.consumers)
    if pg is not None:
        # the frame's gradient row up, the gather-fold over all ranks, the
        # folded vector down (pinned buffers, the library's stream)
        ex = pg.exchange(ctx, 1, n_grad, dev)
        row_h = torch.empty((1, n_grad), dtype=torch.float64).pin_memory()
        row_d = torch.empty((1, n_grad), dtype=torch.float64, device=dev)
        fold_d = torch.empty(n_grad, dtype=torch.float64, device=dev)
        fold_h = torch.empty(n_grad, dtype=torch.float64).pin_memory()

    def exchange(grad_arrays):
        if pg is not None:
            row_h[0].numpy()[:] = np.concatenate(grad_arrays)
            with torch.cuda.stream(stream):
                row_d.copy_(row_h, non_blocking=True)
                ex(row_d, fold_d)
                fold_h.copy_(fold_d, non_blocking=True)
            stream.synchronize()

    def submit(i):
        t, n, _g = tables[i % 2]
        q.check(L.qfb_quant_pass_host_submit(ctx.handle, prec, t, n, ctypes.byref(cfg), i % 2))

    def wait(i):
        q.check(L.qfb_quant_pass_host_wait(ctx.handle, i % 2))
        exchange(tables[i % 2][2])

    for i in range(2):  # warm both slots (their device buffers are sized on first use)
        submit(i)
    for i in range(2):
        wait(i)
    if pg is not None:
        pg.barrier()
    torch.cuda.synchronize(dev)
    k = max(3, args.e2e_steps)
    t0 = time.perf_counter()
    for i in range(k):
        submit(i)
        if i > 0:
            wait(i - 1)
    wait(k - 1)
    torch.cuda.synchronize(dev)
    ms = (time.perf_counter() - t0) * 1e3
    if pg is not None:
        ms = pg.max(ms)
    h2d = sum(p.numel * 4 for p in fp.points) + sum(p.numel * 4 for (p, _c) in fp.consumers)
    d2h = sum(p.numel * 4 * 2 + p.channels * 8 for (p, _c) in fp.consumers)
    if pg is not None:
        h2d += 8 * n_grad
        d2h += 8 * n_grad
    return {"value": ws * k / (ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": k,
            "timing": "host wall clock around the submit/wait calls (the pass is synchronous per "
                      "frame: wait returns when the outputs are in host memory), max over ranks",
            "api": "qfb_quant_pass_host_submit/_wait (one pair per frame: 19 tensors, 22 quant points; "
                   "float32 pinned host buffers" + ("; EmulatedHalf precision: values on the binary16 grid, "
                                                    "half-grid FQ outputs" if args.dtype == "f16" else "") +
                   "; H2D/compute/D2H pipelined per point, two frames in flight" +
                   ("; + per frame the gradient row exchange (up, NCCL gather-fold, down)" if pg is not None
                    else "") + ")"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_qfb(args)


if __name__ == "__main__":
    sys.exit(main())
