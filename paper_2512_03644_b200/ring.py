"""Host-side wiring of the DP-ring replicas across ranks (plumbing).

One process per GPU.  Every rank holds the replica of its ring predecessor
(reference SPEC.md:516-517, controller.cpp:179-180: the replica of
(dp, pp, tp) lives on (dp+1 mod d, pp, tp)) and snapshots into the replica
its successor holds.  Replica memory is exported as an opaque handle
(ffx_replica_export: CUDA IPC + layout) and exchanged with
torch.distributed's object collectives; the data path itself never touches
the host.

The functions take the export / open / all-gather operations as arguments so
the wiring is testable on CPU with gloo (tests/test_ring_wiring.py).
"""
from __future__ import annotations

from typing import Callable, List, Sequence


def ring_roles(world: int, p: int = 1, t: int = 1):
    """Global index -> (dp, pp, tp), tensor fastest, then pipeline, then data
    parallel (reference domain.cpp:18-30)."""
    return [(i // (t * p), (i // t) % p, i % t) for i in range(world)]


def successor(rank: int, world: int, p: int = 1, t: int = 1, k: int = 1) -> int:
    """Rank holding this rank's k-th replica: (dp+k mod d, pp, tp)."""
    d = world // (p * t)
    dp, pp, tp = ring_roles(world, p, t)[rank]
    return (((dp + k) % d) * p + pp) * t + tp


def predecessor(rank: int, world: int, p: int = 1, t: int = 1, k: int = 1) -> int:
    d = world // (p * t)
    dp, pp, tp = ring_roles(world, p, t)[rank]
    return (((dp - k) % d) * p + pp) * t + tp


def wire_ring(rank: int, world: int, create_for: Callable[[int], object], export: Callable[[object], bytes],
              open_handle: Callable[[bytes], object], all_gather: Callable[[bytes], List[bytes]],
              p: int = 1, t: int = 1, replicas: int = 1):
    """Create the replicas this rank holds, exchange handles, open the ones
    this rank writes into.

    Returns (held, targets, handles):
      held[k]    replica this rank holds for predecessor k+1 steps back
      targets[k] opened view of the replica that successor k+1 holds for us
      handles[r][k] every rank's exported handle (needed again for recovery)
    """
    held = [create_for(predecessor(rank, world, p, t, k + 1)) for k in range(replicas)]
    mine = b"".join(export(h) for h in held)
    gathered = all_gather(mine)
    hb = len(mine) // replicas if replicas else 0
    handles = [[g[i * hb:(i + 1) * hb] for i in range(replicas)] for g in gathered]
    targets = [open_handle(handles[successor(rank, world, p, t, k + 1)][k]) for k in range(replicas)]
    return held, targets, handles


def recovery_sources(plan_forwards: Sequence, world: int, p: int = 1, t: int = 1):
    """Map plan_recovery forwards (origin Role, holder_node, dest_node,
    holder_dp) to (origin rank, holder rank, replica index k) so the
    replacement knows which exported handle to open."""
    out = []
    d = world // (p * t)
    for origin, _hn, _dn, holder_dp in plan_forwards:
        o = origin.tuple() if hasattr(origin, "tuple") else tuple(origin)
        origin_rank = (o[0] * p + o[1]) * t + o[2]
        holder_rank = (holder_dp * p + o[1]) * t + o[2]
        k = (holder_dp - o[0]) % d - 1
        out.append((origin_rank, holder_rank, k))
    return out


class WiringError(RuntimeError):
    """A step failed on some rank; every rank raises it at the same point, so
    no rank is left waiting in a collective (or in a multicast bind, which
    blocks until every member joined)."""


def _agree(all_gather, ok: bool, what: str, err: str = ""):
    results = all_gather((bool(ok), err))
    bad = [(i, e) for i, (o, e) in enumerate(results) if not o]
    if bad:
        raise WiringError("%s failed on ranks %s: %s" % (what, [i for i, _ in bad], bad[0][1]))


def wire_mcast_ring(rank: int, world: int, create_for: Callable[[int], object], export: Callable[[object], bytes],
                    open_handle: Callable[[bytes], object], create_mcast: Callable[[], object],
                    export_mcast: Callable[[object], bytes], open_mcast: Callable[[bytes], object],
                    all_gather: Callable[[bytes], List[bytes]], barrier: Callable[[], None],
                    p: int = 1, t: int = 1, replicas: int = 2):
    """Double neighbour over NVSwitch multicast: rank r's
    snapshot goes ONCE into a multicast range bound to the replicas its
    successors 1..replicas hold for it.

    Every rank: creates the (shareable) replicas it holds for its
    predecessors 1..replicas and its own multicast object; handles are
    all-gathered; it opens the multicast objects of its predecessors; every
    member joins every team it is in (barrier) before any bind; holders bind;
    the origin opens its first holder's replica as the read view.  Each
    phase ends with an agreement round: a failure anywhere raises
    WiringError on every rank (objects created so far are returned through
    the exception's `created` attribute for cleanup).

    Returns (held, own_mc, pred_mcs, view, handles) -- handles[r][k] as in
    wire_ring, so recovery_sources() applies unchanged; the caller makes
    own_mc + view its snapshot target (ffx_snapshot_target_mcast).
    """
    created = {"held": [], "own": None, "preds": [], "view": None}

    def phase(what, fn):
        err, ok = "", True
        try:
            fn()
        except Exception as ex:  # reported collectively below
            ok, err = False, repr(ex)
        try:
            _agree(all_gather, ok, what, err)
        except WiringError as ex:
            ex.created = created
            raise

    def make():
        for k in range(replicas):
            created["held"].append(create_for(predecessor(rank, world, p, t, k + 1)))
        created["own"] = create_mcast()

    phase("replica / multicast creation", make)
    held, own = created["held"], created["own"]
    mine = (b"".join(export(h) for h in held), export_mcast(own))
    gathered = all_gather(mine)
    hb = len(mine[0]) // replicas if replicas else 0
    handles = [[g[0][i * hb:(i + 1) * hb] for i in range(replicas)] for g in gathered]

    def join():
        for k in range(replicas):
            created["preds"].append(open_mcast(gathered[predecessor(rank, world, p, t, k + 1)][1]))
        for m in [own] + created["preds"]:
            m.join()

    phase("multicast join", join)
    barrier()  # every team complete before anyone binds or maps
    preds = created["preds"]

    def bind():
        for m, h in zip(preds, held):
            m.bind(h)
        created["view"] = open_handle(handles[successor(rank, world, p, t, 1)][0])

    phase("multicast bind", bind)
    return held, own, preds, created["view"], handles
