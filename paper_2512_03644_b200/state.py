"""State-registry layouts of the BASELINE configs and their synthetic content.

Sizes follow the reference's sizing rules exactly (size table):
  unique optimizer bytes per DP rank = ceil(12 phi / d) when the optimizer is
  distributed and d > 1 (evo::optimizer_bytes, evolution.cpp:15-19; razor,
  ckpt.cpp:13-21), and the bf16 parameter shard a ZeRO-3 rank owns is
  ceil(2 phi / d) (SURVEY 7.2 hard part 8: unique under ZeRO-3).

A ZeRO-3 rank registers six regions (the north star's "fp32/bf16 master
params, Adam m/v, data-loader cursor and RNG state"):
  MASTER fp32 ceil(4phi/d) | ADAM_M ceil(4phi/d) | ADAM_V (the rest of ceil(12phi/d))
  | PARAMS bf16 ceil(2phi/d) | CURSOR 16 B | RNG 16 B
so MASTER + ADAM_M + ADAM_V is exactly the reference's unique payload and the
Llama-3 8B d=8 shard is 12,045,391,872 + 2,007,565,312 + 32 bytes.

Content is synthetic and checkable: every large region is
evo::materialize(key, bytes) (evolution.cpp:88-97; generated on the device by
ffx.materialize) for a 32-byte key hashed the reference's way (HashIn,
hash.cpp:52-100: every field little-endian, strings length-prefixed), so
restored regions can be checked with blob_is_sound and against the oracle's
materialize_range.  The cursor is (iteration, dp) and the RNG word
(seed, philox offset), as 2 x u64 LE each.

No oracle import here: the keys are product-side (hashlib), pinned to the
oracle by tests/test_state_layout.py.
"""
from __future__ import annotations

import hashlib
import struct
from dataclasses import dataclass
from typing import List, Optional

# parameters per model (SURVEY 8 sizes)
PHI_GPT2_SMALL = 124_439_808
PHI_GPT2_XL = 1_557_611_200
PHI_LLAMA3_8B = 8_030_261_248
PHI_LLAMA3_70B = 70_553_706_496

# ffx_region_kind (include/ffx.h)
MASTER, ADAM_M, ADAM_V, PARAMS, CURSOR, RNG, BLOB = range(7)


class HashIn:
    """ftsim::HashIn (hash.cpp:52-100): LE fields, length-prefixed strings."""

    def __init__(self):
        self._b = bytearray()

    def str(self, s: str) -> "HashIn":
        b = s.encode()
        self._b += struct.pack("<Q", len(b)) + b
        return self

    def u64(self, v: int) -> "HashIn":
        self._b += struct.pack("<Q", v & 0xFFFFFFFFFFFFFFFF)
        return self

    def u32(self, v: int) -> "HashIn":
        self._b += struct.pack("<I", v & 0xFFFFFFFF)
        return self

    def u16(self, v: int) -> "HashIn":
        self._b += struct.pack("<H", v & 0xFFFF)
        return self

    def digest(self) -> bytes:
        return hashlib.sha256(bytes(self._b)).digest()


def optimizer_init(seed: int, dp: int, pp: int, tp: int, distributed: bool = True) -> bytes:
    """evo::optimizer_init (evolution.cpp:25-31)."""
    h = HashIn().str("O0").u64(seed)
    if distributed:
        h.u16(dp)
    return h.u16(pp).u16(tp).digest()


def weights_init(seed: int, pp: int, tp: int) -> bytes:
    """evo::weights_init (evolution.cpp:21-23)."""
    return HashIn().str("W0").u64(seed).u16(pp).u16(tp).digest()


def optimizer_bytes(phi: int, d: int, distributed: bool = True) -> int:
    """evo::optimizer_bytes (evolution.cpp:15-19)."""
    full = 12 * phi
    return full if (not distributed or d <= 1) else (full + d - 1) // d


def region_key(seed: int, dp: int, kind: int, iteration: int) -> bytes:
    """Key of one synthetic region of rank dp at an iteration (a HashIn in the
    reference's style; the "R" tag keeps it apart from the reference's own
    weights / optimizer keys)."""
    return HashIn().str("R").u64(seed).u16(dp).u16(0).u16(0).u32(kind).u64(iteration).digest()


@dataclass
class Region:
    kind: int
    nbytes: int
    digest: Optional[bytes] = None   # materialize(digest, nbytes)
    literal: Optional[bytes] = None  # exactly these bytes

    def spec(self) -> str:
        """ffx_standby's region syntax (kind:bytes:HEX64 | kind:bytes:=HEX)."""
        if self.literal is not None:
            return "%d:%d:=%s" % (self.kind, self.nbytes, self.literal.hex())
        return "%d:%d:%s" % (self.kind, self.nbytes, self.digest.hex())


def zero3_shard(phi: int, d: int, dp: int, seed: int = 42, iteration: int = 1) -> List[Region]:
    """The six regions a ZeRO-3 DP rank registers (module docstring)."""
    unique = optimizer_bytes(phi, d, True)
    quarter = (4 * phi + d - 1) // d
    sizes = [(MASTER, quarter), (ADAM_M, quarter), (ADAM_V, unique - 2 * quarter),
             (PARAMS, (2 * phi + d - 1) // d)]
    out = [Region(k, n, digest=region_key(seed, dp, k, iteration)) for k, n in sizes]
    out.append(Region(CURSOR, 16, literal=struct.pack("<QQ", iteration, dp)))
    out.append(Region(RNG, 16, literal=struct.pack("<QQ", seed, iteration * 4096)))
    return out


def shard_bytes(regions: List[Region]) -> int:
    return sum(r.nbytes for r in regions)


def allocate(ffx, torch, ctx, regions: List[Region], device=None):
    """Allocate, fill (on the device) and register the regions; returns the
    tensors in registration order."""
    out = []
    for r in regions:
        t = torch.empty(r.nbytes, dtype=torch.uint8, device=device or "cuda")
        fill(ffx, torch, t, r)
        ctx.register(r.kind, t)
        out.append(t)
    return out


def fill(ffx, torch, t, r: Region):
    if r.literal is not None:
        t.copy_(torch.frombuffer(bytearray(r.literal), dtype=torch.uint8))
    else:
        ffx.materialize(t, r.digest)
