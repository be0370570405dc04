// test_facade_device.cpp -- the reference API driven with DEVICE state.
//
// The reference's HostSnapshots::take(it, ptr, len) (ckpt.cpp:38-53) takes a
// host pointer; the B200 facade also accepts device pointers and then
// snapshots the live HBM state in place (no staging copy).  This checks that
// path end to end against the same API's host-pointer behaviour:
//   device state -> HostSnapshots::take -> framed() == pack_blob(host copy)
//   -> NeighborBuffer::store -> framed_at() -> assemble_restore -> bytes equal.
// Built by paper_2512_03644_b200/facade/Makefile, run by
// tests/test_gpu_reference_suite.py on the GPU box.
#include <cstdio>
#include <cstring>
#include <vector>

#include "ffx.h"
#include "ftsim/ckpt.hpp"
#include "ftsim/evolution.hpp"
#include "ftsim/hash.hpp"
#include "ftsim/storage.hpp"

using namespace ftsim;

static int failures = 0;
#define EXPECT(c)                                                     \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "%s:%d: FAILED %s\n", __FILE__, __LINE__, #c); \
      ++failures;                                                     \
    }                                                                 \
  } while (0)

int main() {
  const Role me{1, 0, 0}, peer{0, 0, 0};
  const std::uint64_t n = (1u << 22) + 77;
  const Digest d = evo::optimizer_init(42, me, true);

  void* dev = nullptr;
  if (ffx_device_alloc(0, n, &dev) != FFX_OK) {
    std::fprintf(stderr, "no device: %s\n", ffx_last_error());
    return 2;
  }
  EXPECT(ffx_materialize(dev, d.data(), n, nullptr) == FFX_OK);
  std::vector<std::uint8_t> host(n);
  EXPECT(ffx_memcpy(host.data(), dev, n, nullptr, 1) == FFX_OK);
  EXPECT(host == evo::materialize(d, n));
  EXPECT(evo::blob_is_sound(host));

  // take() from device memory == framing the host copy
  ckpt::HostSnapshots hs(me, n);
  hs.take(9, dev, n);
  hs.take(10, dev, n);
  const auto* f10 = hs.framed(10);
  EXPECT(f10 != nullptr);
  EXPECT(*f10 == store::pack_blob(me, 10, store::BlobKind::Optimizer, host));
  EXPECT(hs.previous().value() == 9);
  EXPECT(checksum64(dev, n) == checksum64(host));

  // holder side validates and keeps it; restore reassembles it
  ckpt::NeighborBuffer nb(me);
  nb.store(*f10);
  EXPECT(nb.newest().value() == 10);
  ClusterSpec cs;
  cs.num_nodes = 1;
  cs.gpus_per_node = 2;
  cs.data_parallel = 2;
  cs.params_per_device = 64;
  cs.distributed_optimizer = true;
  const auto plan = ckpt::razor(cs);
  const auto weights = store::pack_blob(peer, 10, store::BlobKind::Weights,
                                        evo::materialize(evo::weights_init(42, me), 128));
  ckpt::RestorePieces pieces;
  pieces.unique = nb.framed_at(10);
  pieces.weights = &weights;
  const StateBundle b = ckpt::assemble_restore(me, 10, plan, pieces);
  EXPECT(b.optimizer_current.blob == host);
  EXPECT(b.iteration == 10);

  // a flipped byte in the device state changes the snapshot checksum
  std::uint8_t one = 0;
  EXPECT(ffx_memcpy(&one, static_cast<std::uint8_t*>(dev) + 12345, 1, nullptr, 1) == FFX_OK);
  one ^= 0x5A;
  EXPECT(ffx_memcpy(static_cast<std::uint8_t*>(dev) + 12345, &one, 1, nullptr, 1) == FFX_OK);
  hs.take(11, dev, n);
  EXPECT(!evo::blob_is_sound(store::unpack_blob(*hs.framed(11)).payload));
  bool threw = false;
  try {
    hs.take(12, dev, n + 1);
  } catch (const ckpt::ConfigError&) {
    threw = true;
  }
  EXPECT(threw);

  // re-taking the OLDER held iteration keeps insertion order (ckpt.cpp:46-52):
  // take(1) take(2) take(1) take(3) holds {2, 3}; framed(2) must still exist
  {
    const std::uint64_t m = 4096 + 5;
    ckpt::HostSnapshots hs2(me, m);
    std::vector<std::uint8_t> a(m, 1), b(m, 2), a2(m, 11), c(m, 3);
    hs2.take(1, a);
    hs2.take(2, b);
    hs2.take(1, a2);
    EXPECT(hs2.newest().value() == 2);
    EXPECT(hs2.previous().value() == 1);
    EXPECT(hs2.framed(1) && *hs2.framed(1) == store::pack_blob(me, 1, store::BlobKind::Optimizer, a2));
    hs2.take(3, c);
    EXPECT(hs2.framed(1) == nullptr);
    EXPECT(hs2.framed(2) && *hs2.framed(2) == store::pack_blob(me, 2, store::BlobKind::Optimizer, b));
    EXPECT(hs2.framed(3) && *hs2.framed(3) == store::pack_blob(me, 3, store::BlobKind::Optimizer, c));
    EXPECT(hs2.newest().value() == 3);
    ckpt::NeighborBuffer nb2(me);
    nb2.store(store::pack_blob(me, 1, store::BlobKind::Optimizer, a));
    nb2.store(store::pack_blob(me, 2, store::BlobKind::Optimizer, b));
    nb2.store(store::pack_blob(me, 1, store::BlobKind::Optimizer, a2));
    EXPECT(nb2.newest().value() == 2);
    nb2.store(store::pack_blob(me, 3, store::BlobKind::Optimizer, c));
    EXPECT(nb2.framed_at(1) == nullptr);
    EXPECT(nb2.framed_at(2) && *nb2.framed_at(2) == store::pack_blob(me, 2, store::BlobKind::Optimizer, b));
    EXPECT(nb2.newest().value() == 3);
  }

  ffx_device_free(0, dev);
  std::printf("[facade-device] %s (%d failures)\n", failures ? "FAILED" : "ok", failures);
  return failures ? 1 : 0;
}
