"""A real training loop survives a failure: the per-iteration snapshot of its
ZeRO-style flat state (fp32 master weights, Adam m and v, the data cursor /
step counter) lands in the neighbour's replica, the state is destroyed after
iteration 5, restored from the replica, and training continues -- the loss
trajectory afterwards is bit-identical to an uninterrupted run.

The reference models the state as synthetic blobs (evolution.cpp); this is
the same path (register regions -> snapshot per iteration -> recover) on
tensors an optimizer actually mutates."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

IN, HID, OUT, BATCH = 256, 512, 10, 64
SHAPES = [(IN, HID), (HID,), (HID, OUT), (OUT,)]
NPARAM = sum(torch.Size(s).numel() for s in SHAPES)


@pytest.fixture(scope="module")
def ffx():
    from paper_2512_03644_b200 import ffx as m
    return m


class Trainer:
    """2-layer MLP whose parameters are views of one flat fp32 buffer (the
    ZeRO flat partition); Adam written out over flat m / v buffers."""

    def __init__(self, seed=1):
        g = torch.Generator(device="cuda").manual_seed(seed)
        self.flat = (torch.randn(NPARAM, device="cuda", generator=g) * 0.05).requires_grad_(True)
        self.m = torch.zeros(NPARAM, device="cuda")
        self.v = torch.zeros(NPARAM, device="cuda")
        self.cursor = torch.zeros(2, dtype=torch.int64, device="cuda")  # [step, data position]

    def params(self):
        out, o = [], 0
        for s in SHAPES:
            n = torch.Size(s).numel()
            out.append(self.flat[o:o + n].view(s))
            o += n
        return out

    def batch(self):
        pos = int(self.cursor[1].item())
        g = torch.Generator(device="cuda").manual_seed(1000 + pos)
        x = torch.randn(BATCH, IN, device="cuda", generator=g)
        y = torch.randint(0, OUT, (BATCH,), device="cuda", generator=g)
        return x, y

    def step(self, lr=1e-3, b1=0.9, b2=0.999, eps=1e-8):
        x, y = self.batch()
        w1, c1, w2, c2 = self.params()
        loss = torch.nn.functional.cross_entropy(torch.relu(x @ w1 + c1) @ w2 + c2, y)
        self.flat.grad = None
        loss.backward()
        with torch.no_grad():
            t = int(self.cursor[0].item()) + 1
            gr = self.flat.grad
            self.m.mul_(b1).add_(gr, alpha=1 - b1)
            self.v.mul_(b2).addcmul_(gr, gr, value=1 - b2)
            mh = self.m / (1 - b1 ** t)
            vh = self.v / (1 - b2 ** t)
            self.flat.sub_(lr * mh / (vh.sqrt() + eps))
            self.cursor += 1
        return loss.detach().clone()

    def regions(self):
        return [self.flat.detach(), self.m, self.v, self.cursor]


def test_training_resumes_bit_exact_after_recovery(ffx):
    torch.backends.cuda.matmul.allow_tf32 = False
    ref = Trainer()
    ref_losses = [ref.step() for _ in range(10)]

    run = Trainer()
    spec = ffx.make_spec(d=2, phi=NPARAM, distributed=True)
    holder = ffx.Context(0, spec, (1, 0, 0))
    me = ffx.Context(0, spec, (0, 0, 0))
    kinds = [ffx.REGION_MASTER, ffx.REGION_ADAM_M, ffx.REGION_ADAM_V, ffx.REGION_CURSOR]
    for k, t in zip(kinds, run.regions()):
        me.register(k, t)
    nbytes = sum(t.numel() * t.element_size() for t in run.regions())
    rep = holder.create_replica((0, 0, 0), nbytes + 4096, 2)
    view = me.open_replica(rep.export())
    me.set_target(view)
    try:
        losses = []
        for it in range(1, 6):
            losses.append(run.step())
            me.snapshot(it)  # after the optimizer update of iteration `it`
        torch.cuda.synchronize()
        assert rep.newest() == 5
        # the rank dies: every byte of its training state is gone
        me.inject(ffx.FAULT_POISON_STATE)
        torch.cuda.synchronize()
        assert not torch.equal(run.m, ref.m)
        rpt = me.recover(view, 5)
        assert rpt.bad_slices == 0 and rpt.bytes == nbytes
        assert int(run.cursor[0].item()) == 5
        for _ in range(5):
            losses.append(run.step())
        for a, b in zip(losses, ref_losses):
            assert torch.equal(a, b)  # bit-identical trajectory
        assert torch.equal(run.flat.detach(), ref.flat.detach())
        assert torch.equal(run.m, ref.m) and torch.equal(run.v, ref.v)
    finally:
        torch.cuda.synchronize()
        view.destroy()
        rep.destroy()
        me.close()
        holder.close()
