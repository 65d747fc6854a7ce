"""Asynchronous update scheme (PAPER.md:266-282 [Sec. 5.1], Fig. 5): the buffers
and the scheduler around the library's per-side steps.

Every step of the path runs in libparagan's kernels (paragan_d_step_fakes, paragan_g_step,
paragan_generate, paragan_export_fakes / _state, paragan_import_state); this module only moves
device buffers between them — img_buff (generated batches, G -> D) and the D snapshots G trains
through (D -> G) — and decides which entry each side consumes (R31-R33):

  * tick t, D side: n_d D steps, each on the oldest img_buff entry whose tag (the tick of the G
    version that produced it) satisfies t - tag <= max_staleness; when none is left (cold start, or
    max_staleness = 0) the current G generates one (tag t);
  * tick t, G side: one G step through the D snapshot tagged t - max_staleness (D after that tick's
    D update; the initial D at cold start), imported into the G context as a copy; its fakes (tag t)
    go to img_buff, split into g_batch / d_batch entries ("possible to apply different batch sizes for
    both parties").

Two drivers with the same semantics:
  * ``LocalAsync``: both sides in one process (two contexts on one GPU), deterministic interleaving —
    the parity configuration (max_staleness = 0 reproduces the synchronous iteration);
  * ``DistributedAsync``: G and D on disjoint GPU groups of one box ("run both generator and
    discriminator in parallel on different nodes"), each group data-parallel with its own NCCL
    communicator inside the library; at each tick boundary G rank i and D rank i exchange the previous
    tick's fakes and D snapshot with one batched NCCL send/recv pair (torch.distributed, plumbing), so
    both sides compute concurrently with staleness exactly max_staleness = 1.
"""
from __future__ import annotations

from collections import deque

from . import api


class StaleBufferError(RuntimeError):
    pass


class ImageBuffer:
    """img_buff: bounded FIFO of (fakes, labels, tag); drop-oldest on overflow (evictions counted)."""

    def __init__(self, capacity: int):
        assert capacity >= 1
        self.capacity, self.q, self.evicted, self.produced, self.consumed, self.stale_dropped = capacity, deque(), 0, 0, 0, 0

    def push(self, fakes, labels, tag: int):
        if len(self.q) == self.capacity:
            self.q.popleft()
            self.evicted += 1
        self.q.append((fakes, labels, tag))
        self.produced += 1

    def pop(self, now: int, max_staleness: int):
        """The oldest entry with now - tag <= max_staleness (older ones are dropped); None when empty."""
        while self.q and now - self.q[0][2] > max_staleness:
            self.q.popleft()
            self.stale_dropped += 1
        if not self.q:
            return None
        self.consumed += 1
        return self.q.popleft()

    def __len__(self):
        return len(self.q)


class SnapshotBuffer:
    """pred_buff's role on this path: D states G may train through, tagged by the tick after whose D update
    they were taken (-1 = the initial D)."""

    def __init__(self):
        self.q = []

    def push(self, state, tag: int):
        self.q.append((state, tag))

    def select(self, now: int, max_staleness: int):
        want = now - max_staleness
        cand = [s for s in self.q if s[1] <= want]
        state, tag = cand[-1] if cand else self.q[0]
        self.q = [s for s in self.q if s[1] >= tag]   # older snapshots are never needed again
        return state, now - tag


class LocalAsync:
    """Both sides on one device: ctx_g (G + a D snapshot) and ctx_d (the live D)."""

    def __init__(self, cfg_g, cfg_d, max_staleness: int = 1, capacity: int = 4, stream=None):
        import torch
        assert cfg_g.local_batch % cfg_d.local_batch == 0, "g_batch must be a multiple of d_batch"
        self.s, self.cfg_g, self.cfg_d = max_staleness, cfg_g, cfg_d
        self.ctx_g = api.Context(cfg_g, stream=stream)
        self.ctx_d = api.Context(cfg_d, stream=stream)
        self.dev = f"cuda:{cfg_g.device}"
        self.tdt = torch.bfloat16 if cfg_g.compute == api.BF16 else torch.float32
        self.img_buff = ImageBuffer(capacity)
        self.snaps = SnapshotBuffer()
        self.ticks = 0

    def set_params(self, g_flat, d_flat):
        self.ctx_g.set_params(api.NET_G, g_flat)
        self.ctx_g.set_params(api.NET_D, d_flat)
        self.ctx_d.set_params(api.NET_D, d_flat)
        self.ctx_d.set_params(api.NET_G, g_flat)
        self.snaps = SnapshotBuffer()
        self.snaps.push(self._state(self.ctx_d), -1)

    def _state(self, ctx):
        import torch
        buf = torch.empty(ctx.state_size(api.NET_D), dtype=torch.float32, device=self.dev)
        ctx.export_state(api.NET_D, buf)
        return buf

    def _images(self, n):
        import torch
        r = self.cfg_g.resolution
        return torch.empty((n, r, r, self.cfg_g.c_pad_image), dtype=self.tdt, device=self.dev)

    def tick(self, d_batches, g_batch):
        """d_batches: [(real_nhwc, real_y, z_boot, y_boot)] * n_d (device tensors); g_batch: (z, y)."""
        import torch
        t = self.ticks
        stale = []
        for real, ry, zb, yb in d_batches:
            e = self.img_buff.pop(t, self.s)
            if e is None:   # cold start / max_staleness 0: the current G generates the batch
                f = self._images(self.cfg_d.local_batch)
                self._generate(zb, yb, f)
                e = (f, yb, t)
                self.img_buff.produced += 1
                self.img_buff.consumed += 1
            fakes, fy, tag = e
            self.ctx_d.d_step_fakes(real, ry, fakes, fy)
            stale.append(t - tag)
        self.snaps.push(self._state(self.ctx_d), t)
        snap, g_stale = self.snaps.select(t, self.s)
        self.ctx_g.import_state(api.NET_D, snap)
        z, y = g_batch
        self.ctx_g.g_step(z, y, flags=api.FLAG_ASYNC)
        out = self._images(self.cfg_g.local_batch)
        self.ctx_g.export_fakes(out)
        b = self.cfg_d.local_batch
        for i in range(0, self.cfg_g.local_batch, b):
            self.img_buff.push(out[i:i + b], y[i:i + b], t)
        self.ticks += 1
        return {"d_staleness": stale, "g_snapshot_staleness": g_stale}

    def _generate(self, z, y, dst):
        """A d_batch-sized batch from the current G (the G context's copy of G is the live one)."""
        if self.cfg_g.local_batch == self.cfg_d.local_batch:
            self.ctx_g.generate(z, y, dst)
        else:   # the D context keeps a copy of G (refreshed here) sized for d_batch
            import torch
            buf = torch.empty(self.ctx_g.state_size(api.NET_G), dtype=torch.float32, device=self.dev)
            self.ctx_g.export_state(api.NET_G, buf)
            self.ctx_d.import_state(api.NET_G, buf)
            self.ctx_d.generate(z, y, dst)
            self.ctx_d.export_state(api.NET_G, buf)      # G's u advanced by this forward (R4)
            self.ctx_g.import_state(api.NET_G, buf)

    def close(self):
        self.ctx_g.close()
        self.ctx_d.close()


class DistributedAsync:
    """G on ranks [0, W/2), D on ranks [W/2, W) of one box; G rank i pairs with D rank W/2 + i.
    Staleness is exactly 1: at each tick boundary both sides send last tick's output and receive the
    other side's (one batched NCCL send/recv), then compute concurrently."""

    def __init__(self, make_cfg, g_batch: int, d_batch: int, n_d: int = 1):
        import torch
        import torch.distributed as dist
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        assert self.world % 2 == 0, "needs an even number of ranks (G group + D group)"
        assert g_batch == n_d * d_batch, "each G batch feeds the n_d D steps of the next tick"
        half = self.world // 2
        self.is_g = self.rank < half
        self.grank = self.rank if self.is_g else self.rank - half
        self.peer = self.rank + half if self.is_g else self.rank - half
        groups = [dist.new_group(list(range(half))), dist.new_group(list(range(half, self.world)))]
        self.group = groups[0] if self.is_g else groups[1]
        leader = 0 if self.is_g else half
        obj = [api.get_unique_id() if self.rank == leader else None]
        dist.broadcast_object_list(obj, src=leader, group=self.group)
        self.cfg = make_cfg(g_batch if self.is_g else d_batch, self.grank, half)
        self.stream = torch.cuda.current_stream()
        self.ctx = api.Context(self.cfg, obj[0] if half > 1 else None, stream=self.stream)
        self.dev = f"cuda:{self.cfg.device}"
        self.g_batch, self.d_batch, self.n_d = g_batch, d_batch, n_d
        tdt = torch.bfloat16 if self.cfg.compute == api.BF16 else torch.float32
        r = self.cfg.resolution
        self.fakes = torch.empty((g_batch, r, r, self.cfg.c_pad_image), dtype=tdt, device=self.dev)
        self.labels = torch.zeros(g_batch, dtype=torch.int32, device=self.dev)
        self.snap = torch.empty(self.ctx.state_size(api.NET_D), dtype=torch.float32, device=self.dev)
        self.t = 0

    def init_params(self, attn_gamma=0.1):
        self.ctx.init_params(attn_gamma)   # same seed on every rank: identical G and D everywhere

    def _exchange(self):
        import torch.distributed as dist
        if self.is_g:
            ops = [dist.P2POp(dist.isend, self.fakes, self.peer), dist.P2POp(dist.isend, self.labels, self.peer),
                   dist.P2POp(dist.irecv, self.snap, self.peer)]
        else:
            ops = [dist.P2POp(dist.isend, self.snap, self.peer), dist.P2POp(dist.irecv, self.fakes, self.peer),
                   dist.P2POp(dist.irecv, self.labels, self.peer)]
        for w in dist.batch_isend_irecv(ops):
            w.wait()

    def tick(self, d_batches=None, g_batch=None, boot=None):
        """G ranks pass g_batch = (z, y) (and boot = (z, y) at tick 0); D ranks pass d_batches =
        [(real_nhwc, real_y)] * n_d."""
        if self.t == 0:
            if self.is_g:   # cold start: the initial G fills the first img_buff entry, the initial D is the snapshot
                self.ctx.generate(boot[0], boot[1], self.fakes)
                self.labels.copy_(boot[1])
            else:
                self.ctx.export_state(api.NET_D, self.snap)
        self._exchange()
        if self.is_g:
            self.ctx.import_state(api.NET_D, self.snap)          # D snapshot of the previous tick
            z, y = g_batch
            self.ctx.g_step(z, y, flags=api.FLAG_ASYNC)
            self.ctx.export_fakes(self.fakes)                     # this tick's img_buff entry
            self.labels.copy_(y)
        else:
            for k, (real, ry) in enumerate(d_batches):           # the previous tick's fakes, d_batch at a time
                sl = slice(k * self.d_batch, (k + 1) * self.d_batch)
                self.ctx.d_step_fakes(real, ry, self.fakes[sl], self.labels[sl])
            self.ctx.export_state(api.NET_D, self.snap)
        self.t += 1

    def close(self):
        self.ctx.close()
