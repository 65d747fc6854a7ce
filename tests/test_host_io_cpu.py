"""Host-side system features, no GPU needed: the congestion-aware prefetcher
(paragan_prefetch_*: in-order, loss-free batches from sample shards; readers and queue depth scale up
while the latency window exceeds the threshold and are released when it falls back) and the
shard format."""
import time

import numpy as np
import pytest

from paper_2411_03999_b200 import api


def _shards(tmp_path, sizes, c=3, h=4, w=4):
    rng = np.random.default_rng(0)
    paths, all_im, all_lb = [], [], []
    for i, n in enumerate(sizes):
        im = rng.standard_normal((n, c, h, w)).astype(np.float32)
        lb = rng.integers(0, 1000, n).astype(np.int32)
        p = str(tmp_path / f"s{i}.pgs")
        api.shard_write(p, im, lb)
        paths.append(p)
        all_im.append(im)
        all_lb.append(lb)
    return paths, np.concatenate(all_im), np.concatenate(all_lb)


def test_prefetch_in_order_and_lossless_across_shards(tmp_path):
    paths, im, lb = _shards(tmp_path, [5, 7, 3])      # 15 samples; batch 4 wraps around
    pf = api.Prefetcher(paths, 4, 3, 4, 4, min_workers=2, max_workers=3)
    total = im.shape[0]
    for b in range(9):
        x, y = pf.next()
        idx = (np.arange(4) + 4 * b) % total
        assert np.array_equal(x, im[idx]) and np.array_equal(y, lb[idx]), b
    pf.close()


def test_prefetch_scales_with_latency_and_releases(tmp_path):
    paths, _, _ = _shards(tmp_path, [64])
    pf = api.Prefetcher(paths, 4, 3, 4, 4, min_workers=1, max_workers=4, min_depth=2, max_depth=16, window=4,
                        latency_threshold_ms=15.0, inject_latency_ms=0.0)
    for _ in range(12):
        pf.next()
    s0 = pf.stats()
    assert s0.active_workers == 1 and s0.depth == 2           # fast storage: minimum resources
    pf.set_latency(40.0)                                        # congestion: every read takes > threshold
    for _ in range(24):
        pf.next()
    s1 = pf.stats()
    assert s1.active_workers > 1 and s1.depth > 2 and s1.scale_ups >= 1, (s1.active_workers, s1.depth)
    pf.set_latency(0.0)                                         # congestion over: resources released
    for _ in range(60):
        pf.next()
    s2 = pf.stats()
    assert s2.active_workers < s1.active_workers and s2.depth < s1.depth and s2.scale_downs >= 1
    pf.close()


def test_prefetch_rejects_bad_config_and_missing_shard(tmp_path):
    paths, _, _ = _shards(tmp_path, [4])
    with pytest.raises(api.ParaganError) as e:
        api.Prefetcher(paths, 4, 3, 4, 4, min_workers=3, max_workers=2)
    assert e.value.status == 2
    with pytest.raises(api.ParaganError) as e:
        api.Prefetcher([str(tmp_path / "missing.pgs")], 4, 3, 4, 4)
    assert e.value.status == 4
    with pytest.raises(api.ParaganError) as e:
        api.Prefetcher(paths, 4, 3, 8, 8)          # shape mismatch with the shard header
    assert e.value.status == 4
