"""The data loader's preload buffer in HBM: PreloadBuffer
semantics (dataloader.hpp:45-73, dataloader.cpp:59-82), DataServerStub's
synthetic samples generated on the device (dataloader.cpp:104-127,
evolution.cpp:112-120) and fold_of_blob (dataloader.cpp:150-164), all
compared with the oracle (and the reference's own functions when
oracle/_ref is built); and preloads issued through the slice scheduler's
link-idle gaps, held back while the buffer is full (SPEC preload_loop)."""
import ctypes

import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


@pytest.fixture
def ctx(ffx):
    c = ffx.Context(0, ffx.make_spec(d=2, phi=1000, distributed=True), (0, 0, 0), 4096)
    yield c
    c.close()


def dev_bytes(ptr, n):
    from paper_2512_03644_b200 import ffx
    out = torch.empty(n, dtype=torch.uint8)
    if n:
        ffx.check(ffx.lib.ffx_memcpy(out.data_ptr(), ptr, n, None, 1), "memcpy")
    return bytes(out.numpy().tobytes())


@pytest.mark.parametrize("seed,first,count,sb", [(42, 0, 1, 8), (42, 1000, 32, 8192), (7, 5, 13, 36),
                                                 (9, 3, 7, 4), (1, 0, 0, 64)])
def test_synthetic_window_is_the_data_servers_bytes(ffx, ctx, seed, first, count, sb):
    p = ffx.Preload(ctx, 1 << 26)
    p.fetch_synthetic(3, ffx.data_item_digests(seed, first, count), sb)
    dev, n = p.take(3)
    torch.cuda.synchronize()
    assert n == count * sb
    got = dev_bytes(dev, n)
    want = orc.fetch(seed, first, count, sb)
    assert got == want
    r = orc.ref_lib()
    if r is not None and hasattr(r, "ref_fetch") and n:
        buf = ctypes.create_string_buffer(n)
        r.ref_fetch(seed, first, count, sb, buf)
        assert buf.raw == got
    if n:
        fold = ffx.fold_of_blob(dev, sb, nbytes=n)
        assert fold == orc.fold_of_blob(want, sb)
        if sb >= 8:  # the first 8 bytes of a sample are item_fold(data_item(., 8)): window_fold
            lib = orc.lib
            lib.orc_window_fold.restype = ctypes.c_uint64
            lib.orc_window_fold.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint32]
            assert fold == lib.orc_window_fold(seed, first, count)
    p.free(dev)
    p.destroy()


def test_host_fetch_and_buffer_semantics(ffx, ctx):
    p = ffx.Preload(ctx, 3000)
    blobs = {it: torch.randint(0, 256, (1000,), dtype=torch.uint8).pin_memory() for it in (5, 6, 7, 8)}
    assert p.fits(3000) and not p.fits(3001)
    for it in (6, 5, 7):
        p.fetch_host(it, blobs[it])
    st = p.info()
    assert (st.bytes, st.entries, st.oldest) == (3000, 3, 5)
    with pytest.raises(ffx.ConfigError):  # overflow (std::logic_error in the reference)
        p.fetch_host(8, blobs[8])
    with pytest.raises(ffx.StateError):   # take() of a TID not held -> nullopt
        p.take(8)
    dev, n = p.take(5)
    with pytest.raises(ffx.StateError):   # consumption evicts
        p.take(5)
    assert dev_bytes(dev, n) == bytes(blobs[5].numpy().tobytes())
    p.free(dev)
    p.fetch_host(8, blobs[8])
    with pytest.raises(ffx.StateError):   # duplicate TID
        p.fetch_host(8, blobs[8])
    assert p.info().oldest == 6
    for it in (6, 7, 8):
        dev, n = p.take(it)
        assert dev_bytes(dev, n) == bytes(blobs[it].numpy().tobytes())
        p.free(dev)
    st = p.info()
    assert (st.bytes, st.entries, st.oldest, st.fetched, st.taken) == (0, 0, 2**64 - 1, 4, 4)
    with pytest.raises(ffx.InvalidArgument):
        ffx.fold_of_blob(torch.zeros(10, dtype=torch.uint8, device="cuda"), 4)
    p.destroy()


def test_preloads_ride_the_schedulers_link_idle_gaps(ffx, ctx):
    """Queued preloads are issued at FFX_GAP_LINK_IDLE reports on the
    scheduler's low-priority copy stream, gated on the step's stream, in
    iteration order; a fetch that does not fit waits for room."""
    sb, count = 4 * 256, 8  # seq_len 256: 1 KiB samples, 8 per worker-iteration
    p = ffx.Preload(ctx, 2 * sb * count)  # room for two iterations
    sched = ffx.Sched(ctx, ffx.SCHED_FUSED, link_gaps=2)
    train = torch.cuda.Stream()
    for it in (1, 2, 3):
        sched.preload_synthetic(p, it, ffx.data_item_digests(42, it * count, count), sb)
    assert sched.preload_pending() == 3 and p.info().entries == 0  # nothing before a gap
    # the "GEMM" on the step's stream; the gap is reported after it
    with torch.cuda.stream(train):
        a = torch.randn(2048, 2048, device="cuda")
        for _ in range(4):
            a = a @ a / 2048
    sched.gap(ffx.GAP_LINK_IDLE, train)
    assert sched.preload_pending() == 1 and p.info().entries == 2  # buffer full: 3 stays queued
    consumer = torch.cuda.Stream()
    dev, n = p.take(1, consumer)
    consumer.synchronize()
    assert dev_bytes(dev, n) == orc.fetch(42, 1 * count, count, sb)
    p.free(dev, consumer)
    sched.gap(ffx.GAP_LINK_IDLE, train)
    assert sched.preload_pending() == 0
    for it in (2, 3):
        dev, n = p.take(it, consumer)
        consumer.synchronize()
        assert dev_bytes(dev, n) == orc.fetch(42, it * count, count, sb)
        p.free(dev, consumer)
    torch.cuda.synchronize()
    sched.destroy()
    p.destroy()
