"""Full-state restore (ffx_recover_full): the unique Adam shard from the ring
successor's replica and the redundant bf16 weights from a live DP peer
(ckpt.cpp:140-167, weights piece :150-152), gathered by one kernel, each part
verified against its own source's checksum table."""
import pytest

import pyoracle as orc

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


def host(t):
    return bytes(t.cpu().numpy().tobytes())


def test_full_state_restore_from_holder_and_live_peer(ffx):
    spec = ffx.make_spec(d=2, phi=(1 << 20), distributed=True)
    n_opt = ffx.optimizer_bytes(spec)      # ceil(12 phi / 2)
    n_w = ffx.weights_bytes(spec)          # 2 phi, redundant across dp
    holder = ffx.Context(0, spec, (0, 0, 0))
    me = ffx.Context(0, spec, (1, 0, 0))
    d_opt = orc.optimizer_init(42, 1, 0, 0, True)
    d_w = orc.weights_init(42, 0, 0)
    opt = torch.empty(n_opt, dtype=torch.uint8, device="cuda")
    w = torch.empty(n_w, dtype=torch.uint8, device="cuda")
    ffx.materialize(opt, d_opt)
    ffx.materialize(w, d_w)
    me.register(ffx.REGION_BLOB, opt)
    me.register(ffx.REGION_PARAMS, w, unique=False)
    rep = holder.create_replica((1, 0, 0), n_opt, 2)
    view = me.open_replica(rep.export())
    me.set_target(view)
    me.snapshot(3)
    # the live peer's weights (identical across the DP ring) and its slice table
    peer_w = torch.empty(n_w, dtype=torch.uint8, device="cuda")
    ffx.materialize(peer_w, d_w)
    peer_sums = torch.empty((n_w + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.slice_checksums(peer_w, 4096, peer_sums)
    torch.cuda.synchronize()
    # failure: both the unique shard and the weights are gone
    opt.fill_(0)
    w.fill_(0xFF)
    r = me.recover_full([view], 3, redundant=[(1, peer_w.data_ptr(), peer_sums.data_ptr())])
    assert r.bad_slices == 0 and r.bytes == n_opt + n_w
    assert host(opt) == orc.materialize(d_opt, n_opt)
    assert host(w) == orc.materialize(d_w, n_w)
    # a bad byte in the live peer's weights is caught in the weights part
    peer_w[777] ^= 1
    with pytest.raises(ffx.RestoreError, match="checksum mismatch"):
        me.recover_full([view], 3, redundant=[(1, peer_w.data_ptr(), peer_sums.data_ptr())])
    # registering the wrong region index is refused
    with pytest.raises(ffx.OutOfRange):
        me.recover_full([view], 3, redundant=[(0, peer_w.data_ptr(), peer_sums.data_ptr())])


def test_peer_table_of_another_slice_size_is_refused(ffx):
    """A live peer's table cut at 4 KiB handed to a 2 KiB context would be
    read past its end (it has half the entries): the region carries its
    table's slice size and a mismatch is a ConfigError, not a fault."""
    spec = ffx.make_spec(d=2, phi=(1 << 20), distributed=True)
    n_w = 3 * (1 << 20) + 5
    holder = ffx.Context(0, spec, (0, 0, 0), 2048)
    me = ffx.Context(0, spec, (1, 0, 0), 2048)
    opt = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    w = torch.empty(n_w, dtype=torch.uint8, device="cuda")
    ffx.materialize(opt, orc.optimizer_init(1, 1, 0, 0, True))
    ffx.materialize(w, orc.weights_init(1, 0, 0))
    me.register(ffx.REGION_BLOB, opt)
    me.register(ffx.REGION_PARAMS, w, unique=False)
    rep = holder.create_replica((1, 0, 0), 1 << 20, 2)
    view = me.open_replica(rep.export())
    me.set_target(view)
    me.snapshot(1)
    peer_w = w.clone()
    s4 = torch.empty((n_w + 4095) // 4096, dtype=torch.int64, device="cuda")
    ffx.slice_checksums(peer_w, 4096, s4)
    with pytest.raises(ffx.ConfigError):
        me.recover_full([view], 1, redundant=[(1, peer_w.data_ptr(), s4.data_ptr(), 4096)])
    s2 = torch.empty((n_w + 2047) // 2048, dtype=torch.int64, device="cuda")
    ffx.slice_checksums(peer_w, 2048, s2)
    torch.cuda.synchronize()
    w.fill_(0)
    r = me.recover_full([view], 1, redundant=[(1, peer_w.data_ptr(), s2.data_ptr(), 2048)])
    assert r.bad_slices == 0 and torch.equal(w, peer_w)
    torch.cuda.synchronize()
    view.destroy()
    rep.destroy()
