"""ParaGAN B200 benchmark: BigGAN-128 training throughput (images/s) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl paragan|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

A step is one ParaGAN iteration — the whole hot path of SURVEY §8(a): layout
pack of the real batch (A1), n_d D steps (SN, G forward with cross-replica BN,
D forward over [fake; real], hinge, D backward, gradient all-reduce, Adam) and
one G step — on BigGAN-128 (ch=96, 158.42M parameters) at 256 images per GPU,
bf16 storage with fp32 last layers, synthetic ImageNet-shaped data and
seeded random-init weights.  Weak scaling: per-GPU batch fixed as N grows.

Inputs: a pool of 4 real batches per D step (fp32 NCHW, resident in HBM; drawn
from the run's random-init generator G0 plus pixel noise, so D is not saturated)
and 4 latent batches, cycled; every step's activations (~70 GB) exceed the
126 MB L2, so no explicit flush is needed.  Timing: W untimed iterations, then
`--repeats` (default 3) timed runs of exactly K iterations, each bracketed by a
barrier + device sync with CUDA events on the compute stream, max over ranks;
the median repeat is reported.

`--impl reference` runs the CPU oracle (oracle/, the only reference this
paper-only task has) on the same metric: each step is a bounded sample of the
workload (a 1:1 iteration of BigGAN-128 on one image), timed on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BigGAN-128 images/sec at 1/2/4/8 B200; scaling eff; conv tensor-pipe util %"
UNIT = "images/s"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """Samples SM clocks and throttle reasons through NVML during the timed region."""

    def __init__(self, device: int):
        self.device, self.samples, self.reasons, self.max_mhz = device, [], set(), None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {getattr(pynvml, k): k for k in dir(pynvml) if k.startswith("nvmlClocksThrottleReason")
                     and isinstance(getattr(pynvml, k), int)}

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for bit, nm in names.items():
                            if bit and (r & bit) == bit and nm not in ("nvmlClocksThrottleReasonAll",
                                                                       "nvmlClocksThrottleReasonNone",
                                                                       "nvmlClocksThrottleReasonGpuIdle",
                                                                       "nvmlClocksThrottleReasonApplicationsClocksSetting"):
                                self.reasons.add(nm.replace("nvmlClocksThrottleReason", "").lower())
                    except Exception:
                        pass
                    time.sleep(0.1)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            pass
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=2)

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def cpu_oracle_sample(res=128, batch=1, seed=7):
    """Time the CPU oracle on one 1:1 iteration of BigGAN-128 at `batch` images (bounded sample)."""
    import torch
    from tests import parity as P
    ocfg = P.oracle_config(res, 96, 64, 1000, 128, 20, bf16=True)
    gs, ds, g0, d0, dbs, gb = P.make_inputs(ocfg, batch, seed)
    t = time.perf_counter()
    P.run_oracle(ocfg, gs, ds, g0, d0, dbs, gb)
    dt = time.perf_counter() - t
    return batch / dt, dt, torch.get_num_threads()


def run_reference(args):
    world, rank, _ = _dist()
    if rank != 0:
        return 0
    import torch
    for _ in range(args.warmup):
        cpu_oracle_sample()
    times = []
    for k in range(args.steps):
        _, dt, cores = cpu_oracle_sample(seed=100 + k)
        times.append(dt)
    tot = sum(times)
    value = args.steps * 1 / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "BigGAN-128 ch=96 training iteration (n_d=1 D steps + 1 G step)",
                       "model": "BigGAN-128 ch=96 (158.42M params)", "global_batch": 1, "per_gpu_batch": 1,
                       "seq_len": None, "parallelism": "dp1", "sample": "1 image per step (bounded CPU sample)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "oracle",
                             "sample": "one BigGAN-128 D+G iteration on 1 image per step (fp64 torch CPU oracle)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _traffic():
    """Per-launch DRAM bytes of the conv kernels from the committed ncu launch list (profiles/)."""
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "round*_traffic.json")))
    if not files:
        return {}
    with open(files[-1]) as f:
        d = json.load(f)
    d["source"] = os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__))) + " (ncu launch list, cold cache)"
    return d


def run_async(args):
    """The asynchronous update scheme on N = 2k GPUs: G steps on ranks [0, k),
    D steps on ranks [k, 2k) (paper_2411_03999_b200/async_gan.DistributedAsync), staleness 1, G batch
    --g-batch per G rank, D batch --batch per D rank (n_d = g_batch / d_batch D steps per tick).  Images/s
    counts the images G trains on (k * g_batch per tick); the D side's real images/s is reported next to it."""
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2411_03999_b200 import api, inputs
    from paper_2411_03999_b200.async_gan import DistributedAsync

    world, rank, local = _dist()
    assert world >= 2 and world % 2 == 0, "--async needs an even number of GPUs"
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    dist.init_process_group("nccl", device_id=torch.device(dev))
    R, gb_, db_ = args.res, args.g_batch or args.batch, args.batch
    n_d = gb_ // db_

    def make_cfg(b, r, w):
        return api.make_config(resolution=R, local_batch=b, d_steps_per_g=n_d, compute=api.BF16, rank=r,
                               world_size=w, device=local, seed=1234)

    da = DistributedAsync(make_cfg, gb_, db_, n_d)
    da.init_params(0.1)
    dz = api.dim_z(da.cfg)
    if da.is_g:
        pool = [inputs.latent_batch(3000 + i, inputs.ROLE_Z_G, da.grank, gb_, dz, 1000) for i in range(4)]
        pool = [(torch.from_numpy(z).to(dev), torch.from_numpy(y).to(dev)) for z, y in pool]
    else:
        pool = []
        for i in range(4):
            ent = []
            for k in range(n_d):
                real, ry = inputs.real_batch(3000 + i, da.grank * n_d + k, db_, R, 1000)
                rp = torch.empty((db_, R, R, 8), dtype=torch.bfloat16, device=dev)
                api.layout_pack(torch.from_numpy(real).to(dev), rp, api.BF16, 8)
                ent.append((rp, torch.from_numpy(ry).to(dev)))
            pool.append(ent)

    def tick(i):
        if da.is_g:
            da.tick(g_batch=pool[i % 4], boot=pool[0])
        else:
            da.tick(d_batches=pool[i % 4])

    for i in range(args.warmup):
        tick(i)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(args.steps):
        tick(args.warmup + i)
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    t = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    k = world // 2
    value = k * gb_ * args.steps / (ms / 1000.0)
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                          "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                          "config": {"workload": f"BigGAN-{R} asynchronous update scheme (P:266-282): G on {k} "
                                                 f"GPUs x {gb_}, D on {k} GPUs x {db_} x n_d={n_d}, staleness 1",
                                     "model": f"BigGAN-{R} ch=96", "g_batch_per_gpu": gb_, "d_batch_per_gpu": db_,
                                     "parallelism": f"G dp{k} + D dp{k}"},
                          "d_real_img_per_s": k * db_ * n_d * args.steps / (ms / 1000.0),
                          "note": "a tick = one G step (G group) concurrent with n_d D steps (D group)"}),
              flush=True)
    da.close()
    dist.destroy_process_group()
    return 0


def _tensor_pipe():
    """ncu tensor-pipe utilisation of the profiled conv kernels (profiles/round*_tensor_pipe.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "round*_tensor_pipe.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    conv = {k: v["tensor_pipe_pct"] for k, v in d.items() if isinstance(v, dict) and k.startswith("k_conv")}
    return conv, os.path.relpath(files[-1], ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="paragan", choices=["paragan", "reference"])
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--res", type=int, default=128)
    ap.add_argument("--d-steps", type=int, default=1)
    ap.add_argument("--repeats", type=int, default=3, help="timed repeats of K steps; the median is reported")
    ap.add_argument("--async", dest="async_", action="store_true",
                    help="asynchronous update scheme (P:266-282): G and D on disjoint halves of the GPUs")
    ap.add_argument("--g-batch", type=int, default=0, help="--async: G batch per G rank (default --batch)")
    ap.add_argument("--reals", default="g0", choices=["g0", "uniform"],
                    help="g0: reals from the initial G plus noise (default, D unsaturated); uniform: U(-1,1) noise "
                         "images without the generation pass (profiling runs: fewer launches before the step)")
    ap.add_argument("--trace", type=int, default=0,
                    help="diagnostic: run this many steps from the initial state, print each step's losses, exit")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--compute", default="bf16", choices=["bf16", "f32"],
                    help="Table 3 precision toggle (P:420-434): bf16 tcgen05 path (default, the bench line) or the "
                         "fp32 SIMT parity engine (an ablation line, never the headline)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.async_:
        return run_async(args)
    assert args.warmup >= 3 or os.environ.get("PARAGAN_ALLOW_SHORT_WARMUP"), "timing rules need >= 3 warm-up steps"

    import numpy as np
    import torch
    from paper_2411_03999_b200 import api, inputs

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    dev = f"cuda:{local}"
    nccl_id = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(dev))
        obj = [api.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    B, R = args.batch, args.res
    compute = api.BF16 if args.compute == "bf16" else api.F32
    if compute == api.F32:
        args.no_profile = True          # no tcgen05 launches to bracket: roofline is the bf16 path's
    cfg = api.make_config(resolution=R, local_batch=B, d_steps_per_g=args.d_steps, compute=compute, rank=rank,
                          world_size=world, device=local, seed=1234)
    stream = torch.cuda.Stream(device=dev)
    nd = args.d_steps
    with torch.cuda.stream(stream):
        ctx = api.Context(cfg, nccl_id, stream=stream)
        ctx.init_params(attn_gamma=0.1)
        dz = api.dim_z(cfg)
        tdt = torch.bfloat16 if compute == api.BF16 else torch.float32
        packed = torch.empty((B, R, R, cfg.c_pad_image), dtype=tdt, device=dev)
        # ---- input pool: 4 (real, labels, z) batches per D step and 4 (z, labels) per G step, resident in
        # HBM (this rank's shard).  "Real" images are drawn from the random-init generator G0 the run
        # starts from (independent latents) plus N(0, 0.05^2) pixel noise, clipped to [-1, 1]: D cannot
        # separate them from the fakes trivially, so the hinge stays out of saturation and the timed D
        # backward multiplies real (non-zero) gradients — unlike uniform-noise reals, which D separates
        # within a few steps (d_loss = 0, dlogits = 0).
        lat = [[inputs.latent_batch(1000 + i, inputs.ROLE_Z_D, rank * nd + k, B, dz, 1000) for k in range(nd)]
               for i in range(4)]
        glat = [inputs.latent_batch(1000 + i, inputs.ROLE_Z_G, rank, B, dz, 1000) for i in range(4)]
        state = {net: ctx.get_params(net) for net in (api.NET_D, api.NET_G)}
        noise_rng = np.random.default_rng(77 + rank)
        pool = []
        for i in range(4):
            reals = []
            for k in range(nd):
                if args.reals == "uniform":
                    reals.append(inputs.real_batch(1000 + i, rank * nd + k, B, R, 1000))
                    continue
                zr, yr = inputs.latent_batch(5000 + i, inputs.ROLE_REAL, rank * nd + k, B, dz, 1000)
                seed_img = torch.zeros((B, R, R, cfg.c_pad_image), dtype=tdt, device=dev)
                ctx.d_step(seed_img, torch.from_numpy(yr).to(dev), torch.from_numpy(zr).to(dev),
                           torch.from_numpy(yr).to(dev), flags=api.FLAG_NO_ALLREDUCE | api.FLAG_NO_UPDATE)
                img = ctx.get_fakes() + noise_rng.normal(0.0, 0.05, size=(B, 3, R, R)).astype(np.float32)
                reals.append((np.clip(img, -1.0, 1.0).astype(np.float32), yr))
            ent = dict(d=[], g=None, host=dict(d=[], g=None))
            for k in range(nd):
                real, ry = reals[k]
                z, fy = lat[i][k]
                hb = dict(real=torch.from_numpy(real).pin_memory(), ry=torch.from_numpy(ry).pin_memory(),
                          z=torch.from_numpy(z).pin_memory(), fy=torch.from_numpy(fy).pin_memory())
                ent["host"]["d"].append(hb)
                ent["d"].append({kk: v.to(dev) for kk, v in hb.items()})
            zg, yg = glat[i]
            hg = dict(zg=torch.from_numpy(zg).pin_memory(), yg=torch.from_numpy(yg).pin_memory())
            ent["host"]["g"] = hg
            ent["g"] = {kk: v.to(dev) for kk, v in hg.items()}
            pool.append(ent)
        for net, flat in state.items():      # back to the initial state (u vectors and Adam state too)
            ctx.set_params(net, flat)

        def step(i, src=None):
            p = src if src is not None else pool[i % 4]
            for d in p["d"]:
                api.layout_pack(d["real"], packed, compute, cfg.c_pad_image, stream)
                ctx.d_step(packed, d["ry"], d["z"], d["fy"])
            ctx.g_step(p["g"]["zg"], p["g"]["yg"])

        def barrier():
            torch.cuda.synchronize(dev)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize(dev)

        def max_over_ranks(x):
            t = torch.tensor([x], device=dev)
            if world > 1:
                torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            return float(t.item())

        if args.trace:
            for i in range(args.trace):
                step(i)
                s2 = ctx.sync_stats(raise_nonfinite=False)
                print(json.dumps({"trace_step": i, "d_loss": float(s2.d_loss), "g_loss": float(s2.g_loss)}),
                      flush=True)
            ctx.close()
            return 0
        for i in range(args.warmup):
            step(i)
        st = ctx.sync_stats(raise_nonfinite=False)
        barrier()
        # ---------------- timed region (device-resident inputs): `repeats` x exactly K iterations, each
        # bracketed by barrier + device sync, CUDA events on the compute stream, max over ranks; the
        # reported value is the median repeat
        rep_ms, launches = [], 0
        with ClockSampler(local) as clk:
            for r in range(args.repeats):
                l0 = ctx.kernel_launches()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                for i in range(args.steps):
                    step(i)
                e1.record(stream)
                barrier()
                rep_ms.append(max_over_ranks(e0.elapsed_time(e1)))
                launches = ctx.kernel_launches() - l0
        st = ctx.sync_stats(raise_nonfinite=False)
        ms_max = statistics.median(rep_ms)
        value = world * B * args.steps / (ms_max / 1000.0)

        # ---------------- end-to-end through the public API with host buffers: every step copies its
        # inputs from pinned host memory and reads its losses back (paragan_sync_stats)
        e2e = None
        d_losses, g_losses = [], []
        if not args.no_e2e:
            # pipelined host loop: step i's inputs are copied from pinned host memory on a copy stream into one
            # of two device input sets (while step i - 1 computes), and step i's losses come back through an
            # asynchronous device -> host copy that the host reads after step i + 1 is enqueued; every byte
            # still crosses inside the timed region, and the region ends after the last read
            import ctypes
            dev_sets = [dict(d=[{k: torch.empty_like(v, device=dev) for k, v in pool[0]["host"]["d"][0].items()}
                                for _ in range(nd)],
                             g={k: torch.empty_like(v, device=dev) for k, v in pool[0]["host"]["g"].items()})
                        for _ in range(2)]
            h2d = sum(v.numel() * v.element_size() for hb in pool[0]["host"]["d"] for v in hb.values()) + \
                sum(v.numel() * v.element_size() for v in pool[0]["host"]["g"].values())
            stats_bytes = ctypes.sizeof(api.Stats)
            stat_bufs = [torch.empty(stats_bytes, dtype=torch.uint8).pin_memory() for _ in range(2)]
            copy_stream = torch.cuda.Stream(device=dev)
            ev_in = [torch.cuda.Event() for _ in range(2)]
            ev_done = [torch.cuda.Event() for _ in range(2)]

            def read(j):
                ev_done[j % 2].synchronize()
                s2 = api.Context.read_stats(stat_bufs[j % 2])
                d_losses.append(round(float(s2.d_loss), 5))
                g_losses.append(round(float(s2.g_loss), 5))

            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            n_e2e = args.steps
            for i in range(n_e2e):
                b = i % 2
                hp = pool[i % 4]["host"]
                if i >= 2:
                    copy_stream.wait_event(ev_done[b])          # step i - 2 has finished reading set b
                with torch.cuda.stream(copy_stream):
                    for k in range(nd):
                        for kk, v in hp["d"][k].items():
                            dev_sets[b]["d"][k][kk].copy_(v, non_blocking=True)
                    for kk, v in hp["g"].items():
                        dev_sets[b]["g"][kk].copy_(v, non_blocking=True)
                    ev_in[b].record(copy_stream)
                stream.wait_event(ev_in[b])
                step(i, src=dev_sets[b])
                ctx.stats_async(stat_bufs[b])                  # device -> host copy of the step's losses
                ev_done[b].record(stream)
                if i >= 1:
                    read(i - 1)
            read(n_e2e - 1)
            f1.record(stream)
            barrier()
            ms2 = max_over_ranks(f0.elapsed_time(f1))
            e2e = {"value": world * B * n_e2e / (ms2 / 1000.0), "unit": UNIT,
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(stats_bytes), "steps": n_e2e}
        d_grad_norm = float(np.linalg.norm(ctx.get_grads(api.NET_D).astype(np.float64)))

        # ---------------- roofline pass: the same steps again with every tcgen05 conv launch bracketed
        # by CUDA events (kept out of the timed region above: the events cost ~2% of the step)
        prof = {}
        if not args.no_profile:
            ctx.profile(True)
            for i in range(args.steps):
                step(i)
            ctx.profile(False)
            for kind in (0, 1, 2, 3, 4, 5, 6):
                prof[kind] = ctx.profile_read(kind)
            barrier()

    if rank == 0:
        burst, sustained, hbm, src = _peaks()
        traffic = _traffic()
        roof = None
        if prof:
            n0, t0, f0_ = prof[0]
            n1, t1, f1_ = prof[1]
            ach = (f0_ / (t0 / 1000.0)) / 1e12 if t0 > 0 else 0.0
            roof = {"bound": "tensor", "kernel": "k_conv_fprop (tcgen05 implicit-GEMM conv, fprop+dgrad launches)",
                    "achieved": ach, "peak": sustained, "unit": "TFLOP/s", "frac": ach / sustained,
                    "peak_source": f"bf16_tflops_sustained ({src}); kernel timed inside a long step",
                    "traffic": traffic.get("conv_fprop", {}).get("dram_bytes_per_launch"),
                    "traffic_source": traffic.get("source"), "launches": n0, "kernel_ms_per_step": t0 / args.steps,
                    "share_of_step": (t0 / args.steps) / (ms_max / args.steps),
                    "achieved_executed": (prof[3][2] / (t0 / 1000.0)) / 1e12 if t0 > 0 else 0.0,
                    "frac_executed": ((prof[3][2] / (t0 / 1000.0)) / 1e12) / sustained if t0 > 0 else 0.0,
                    "note": "achieved = algorithmic flops (G's conv1 over the upsampled tensor, SURVEY 8(d)) / time; "
                            "achieved_executed = flops issued to the tensor cores (sub-pixel conv1: 1/2.25 of its "
                            "algorithmic work) / time.  frac can exceed 1: the sub-pixel decomposition does 2.25x "
                            "less work than the conv it is credited with; frac_executed is the tensor-pipe figure",
                    "wgrad": {"achieved": (f1_ / (t1 / 1000.0)) / 1e12 if t1 > 0 else 0.0,
                              "achieved_executed": (prof[4][2] / (t1 / 1000.0)) / 1e12 if t1 > 0 else 0.0,
                              "launches": n1, "ms_per_step": t1 / args.steps}}
            pipe, pipe_src = _tensor_pipe()
            ex = (prof[3][2] + prof[4][2]) / ((t0 + t1) / 1000.0) / 1e12 if (t0 + t1) > 0 else 0.0
            conv_util = {"executed_tflops": ex, "frac_of_sustained_peak": ex / sustained,
                         "algorithmic_tflops": (f0_ + f1_) / ((t0 + t1) / 1000.0) / 1e12 if (t0 + t1) > 0 else 0.0,
                         "note": "all tcgen05 conv launches (fprop, dgrad, wgrad) of the step, CUDA events: flops "
                                 "issued to the tensor cores / time, vs the measured sustained bf16 peak",
                         "ncu_tensor_pipe_pct": pipe, "ncu_source": pipe_src}
            roof["other_kernels_ms_per_step"] = {
                "fused_attention_fwd_bwd": prof[5][1] / args.steps,
                "g_output_layer_fp32_thin": prof[6][1] / args.steps}
            if world > 1:
                n2, t2, b2 = prof[2]
                roof["collectives"] = {"launches_per_step": n2 / args.steps, "ms_per_step": t2 / args.steps,
                                       "bytes_per_step": b2 / args.steps,
                                       "note": "NCCL all-reduces on the compute stream (rank 0), device time"}
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            v, dt, cores = cpu_oracle_sample()
            cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"one BigGAN-128 D+G iteration on 1 image ({dt:.1f} s, fp64 torch CPU oracle)"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": args.compute, "data": "synthetic",
                "config": {"workload": f"BigGAN-{R} ch=96 training iteration (n_d={args.d_steps} D steps + 1 G step)",
                           "repeats": args.repeats,
                           "model": f"BigGAN-{R} ch=96 (158.42M params)" if R == 128 else f"BigGAN-{R} ch=96",
                           "global_batch": world * B, "per_gpu_batch": B, "seq_len": None,
                           "parallelism": f"dp{world}", "l2": "inputs+activations >> 126 MB L2 (no flush needed)",
                           **({"ablation": "Table 3 precision toggle: fp32 SIMT engine (P:420-434)"}
                              if compute == api.F32 else {})},
                "img_per_s_per_gpu": value / world, "real_img_per_s": value * args.d_steps,
                "roofline": roof, "conv_tensor_pipe_util": conv_util if prof else None,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary(),
                "repeats_ms_per_step": [round(m / args.steps, 3) for m in rep_ms],
                "losses": {"d": st.d_loss, "g": st.g_loss, "d_per_step_e2e": d_losses,
                           "g_per_step_e2e": g_losses, "d_grad_norm_last": d_grad_norm,
                           "reals": ("G0(z') + N(0, 0.05^2) noise, clipped (G0 = the run's random-init generator)"
                                     if args.reals == "g0" else "U(-1, 1) noise images")}}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
