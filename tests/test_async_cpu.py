"""Host logic of the asynchronous update scheme (paper_2411_03999_b200/async_gan.py): the
img_buff FIFO (capacity, drop-oldest eviction, staleness filter, production = consumption + eviction +
stale drops + occupancy) and the D-snapshot selection (exactly max_staleness ticks old, the initial D at
cold start)."""
import pytest

from paper_2411_03999_b200.async_gan import ImageBuffer, SnapshotBuffer


def test_image_buffer_fifo_capacity_and_staleness():
    b = ImageBuffer(capacity=2)
    assert b.pop(0, 1) is None
    b.push("f0", "y0", 0)
    b.push("f1", "y1", 1)
    b.push("f2", "y2", 2)          # full: f0 evicted
    assert b.evicted == 1 and len(b) == 2
    assert b.pop(3, 1)[0] == "f2"  # f1 (tag 1) is 2 ticks old at t=3 -> dropped as stale
    assert b.stale_dropped == 1
    assert b.pop(3, 1) is None
    assert b.produced == b.consumed + b.evicted + b.stale_dropped + len(b)


@pytest.mark.parametrize("s", [0, 1, 2])
def test_snapshot_selection_staleness(s):
    sb = SnapshotBuffer()
    sb.push("D_init", -1)
    seen = []
    for t in range(5):
        sb.push(f"D{t}", t)
        state, stale = sb.select(t, s)
        seen.append((state, stale))
        assert stale <= max(s, t + 1) and (stale == s or t - s < -1)
        assert len(sb.q) <= s + 2
    assert seen[-1] == (f"D{4 - s}", s)
    if s == 2:
        assert seen[0] == ("D_init", 1)    # cold start: the oldest available
