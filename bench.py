"""ParaGAN B200 benchmark: BigGAN-128 training throughput (images/s) on 1..8 B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl paragan|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...          (N > 1)

A step is one ParaGAN iteration — the whole hot path of SURVEY §8(a): layout
pack of the real batch (A1), n_d D steps (SN, G forward with cross-replica BN,
D forward over [fake; real], hinge, D backward, gradient all-reduce, Adam) and
one G step — on BigGAN-128 (ch=96, 158.42M parameters) at 256 images per GPU,
bf16 storage with fp32 last layers, synthetic ImageNet-shaped data and
seeded random-init weights.  Weak scaling: per-GPU batch fixed as N grows.

Inputs: a pool of 4 real batches (fp32 NCHW, resident in HBM) and 4 latent
batches, cycled; every step's activations (~70 GB) exceed the 126 MB L2, so no
explicit flush is needed.  Timing: W untimed iterations, barrier + device sync,
CUDA events on the compute stream around exactly K iterations, max over ranks.

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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="paragan", choices=["paragan", "reference"])
    ap.add_argument("--batch", type=int, default=256, help="images per GPU")
    ap.add_argument("--res", type=int, default=128)
    ap.add_argument("--d-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-profile", action="store_true")
    ap.add_argument("--compute", default="bf16", choices=["bf16", "f32"],
                    help="Table 3 precision toggle (P:420-434): bf16 tcgen05 path (default, the bench line) or the "
                         "fp32 SIMT parity engine (an ablation line, never the headline)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
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
    with torch.cuda.stream(stream):
        ctx = api.Context(cfg, nccl_id, stream=stream)
        ctx.init_params(attn_gamma=0.1)
        dz = api.dim_z(cfg)
        # input pool: 4 batches per rank, resident in HBM (this rank's shard of the global batch)
        pool = []
        for i in range(4):
            real, ry = inputs.real_batch(1000 + i, rank, B, R, 1000)
            z, fy = inputs.latent_batch(1000 + i, inputs.ROLE_Z_D, rank, B, dz, 1000)
            zg, yg = inputs.latent_batch(1000 + i, inputs.ROLE_Z_G, rank, B, dz, 1000)
            pool.append(dict(real=torch.from_numpy(real).to(dev), ry=torch.from_numpy(ry).to(dev),
                             z=torch.from_numpy(z).to(dev), fy=torch.from_numpy(fy).to(dev),
                             zg=torch.from_numpy(zg).to(dev), yg=torch.from_numpy(yg).to(dev),
                             host=dict(real=torch.from_numpy(real).pin_memory(), ry=torch.from_numpy(ry).pin_memory(),
                                       z=torch.from_numpy(z).pin_memory(), fy=torch.from_numpy(fy).pin_memory(),
                                       zg=torch.from_numpy(zg).pin_memory(), yg=torch.from_numpy(yg).pin_memory())))
        packed = torch.empty((B, R, R, cfg.c_pad_image),
                             dtype=torch.bfloat16 if compute == api.BF16 else torch.float32, device=dev)

        def step(i, src=None):
            p = src if src is not None else pool[i % 4]
            for _ in range(args.d_steps):
                api.layout_pack(p["real"], packed, compute, cfg.c_pad_image, stream)
                ctx.d_step(packed, p["ry"], p["z"], p["fy"])
            ctx.g_step(p["zg"], p["yg"])

        def barrier():
            torch.cuda.synchronize(dev)
            if world > 1:
                torch.distributed.barrier()
            torch.cuda.synchronize(dev)

        for i in range(args.warmup):
            step(i)
        st = ctx.sync_stats(raise_nonfinite=False)
        barrier()
        # ---------------- timed region (device-resident inputs)
        l0 = ctx.kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            for i in range(args.steps):
                step(i)
            e1.record(stream)
            barrier()
        ms = e0.elapsed_time(e1)
        launches = ctx.kernel_launches() - l0
        st = ctx.sync_stats(raise_nonfinite=False)
        t = torch.tensor([ms], device=dev)
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_max = float(t.item())
        value = world * B * args.steps / (ms_max / 1000.0)

        # ---------------- end-to-end through the public API with host buffers
        e2e = None
        if not args.no_e2e:
            dev_bufs = {k: torch.empty_like(v, device=dev) for k, v in pool[0]["host"].items()}
            h2d = sum(v.numel() * v.element_size() for v in pool[0]["host"].values())
            h2d = h2d + (args.d_steps - 1) * (pool[0]["host"]["real"].numel() * 4)
            stats_bytes = 4 * 4 + 4 + 16
            barrier()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            n_e2e = args.steps
            for i in range(n_e2e):
                hb = pool[i % 4]["host"]
                for k, v in hb.items():
                    dev_bufs[k].copy_(v, non_blocking=True)
                step(i, src=dict(real=dev_bufs["real"], ry=dev_bufs["ry"], z=dev_bufs["z"], fy=dev_bufs["fy"],
                                 zg=dev_bufs["zg"], yg=dev_bufs["yg"]))
                ctx.sync_stats(raise_nonfinite=False)      # device -> host read of the step's losses
            f1.record(stream)
            barrier()
            ms2 = torch.tensor([f0.elapsed_time(f1)], device=dev)
            if world > 1:
                torch.distributed.all_reduce(ms2, op=torch.distributed.ReduceOp.MAX)
            e2e = {"value": world * B * n_e2e / (float(ms2.item()) / 1000.0), "unit": UNIT,
                   "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(stats_bytes), "steps": n_e2e}

        # ---------------- roofline pass: the same steps again with every tcgen05 conv launch bracketed
        # by CUDA events (kept out of the timed region above: the events cost ~2% of the step)
        prof = {}
        if not args.no_profile:
            ctx.profile(True)
            for i in range(args.steps):
                step(i)
            ctx.profile(False)
            for kind in (0, 1, 2, 3, 4):
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
                    "note": "achieved = algorithmic flops (G's conv1 over the upsampled tensor, SURVEY 8(d)) / time; "
                            "achieved_executed = flops issued to the tensor cores (sub-pixel conv1: 1/2.25 of its "
                            "algorithmic work) / time",
                    "wgrad": {"achieved": (f1_ / (t1 / 1000.0)) / 1e12 if t1 > 0 else 0.0,
                              "achieved_executed": (prof[4][2] / (t1 / 1000.0)) / 1e12 if t1 > 0 else 0.0,
                              "launches": n1, "ms_per_step": t1 / args.steps}}
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
                           "model": f"BigGAN-{R} ch=96 (158.42M params)" if R == 128 else f"BigGAN-{R} ch=96",
                           "global_batch": world * B, "per_gpu_batch": B, "seq_len": None,
                           "parallelism": f"dp{world}", "l2": "inputs+activations >> 126 MB L2 (no flush needed)",
                           **({"ablation": "Table 3 precision toggle: fp32 SIMT engine (P:420-434)"}
                              if compute == api.F32 else {})},
                "img_per_s_per_gpu": value / world, "real_img_per_s": value * args.d_steps,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary(), "losses": {"d": st.d_loss, "g": st.g_loss}}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
