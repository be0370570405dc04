// ftsim/ckpt.hpp -- B200 facade: the checkpoint engine's hot path.
//
// Drop-in for proj/include/ftsim/ckpt.hpp.  Same classes, signatures and
// exception types; the storage behind them moves to the GPU:
//   HostSnapshots   two device-resident version slots (an ffx replica on the
//                   caller's GPU); take() accepts host or device pointers and
//                   runs the fused copy + slice-FNV snapshot kernel.
//   NeighborBuffer  the holder-side replica (two device slots), verified on
//                   store exactly like the reference (checksum + identity).
//   framed()/framed_at()  export SNP1 bytes on demand (cached per version).
//   assemble_restore      validates every piece with device checksums.
// The multi-GPU ring (snapshot straight into a peer's replica over NVLink)
// is the C ABI in include/ffx.h; this header keeps the reference's
// single-process contract.
#pragma once

#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <vector>

#include "ftsim/domain.hpp"
#include "ftsim/storage.hpp"

namespace ftsim::ckpt {

struct UniquenessPlan {
  bool weights_redundant = false;
  bool optimizer_redundant = false;
  std::uint64_t unique_bytes_per_device = 0;
};
UniquenessPlan razor(const ClusterSpec& spec);
inline std::uint64_t unique_state_bytes(const UniquenessPlan& p) { return p.unique_bytes_per_device; }

struct LazyKinds {
  bool weights = false;
  bool optimizer = false;
};
LazyKinds lazy_kinds(const UniquenessPlan& plan);

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct VersionError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RestoreError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

int version_for_target(std::uint64_t held_iteration, std::uint64_t target);
inline bool fallback_due(std::uint64_t iteration, std::uint64_t interval) {
  return interval != 0 && iteration % interval == 0;
}

namespace detail {
struct Slots;  // device replica + its per-version frame cache
}

class HostSnapshots {
 public:
  HostSnapshots(Role role, std::uint64_t capacity_bytes);
  ~HostSnapshots();
  HostSnapshots(HostSnapshots&&) noexcept;
  HostSnapshots& operator=(HostSnapshots&&) noexcept;

  void take(std::uint64_t iteration, const void* unique, std::size_t len);
  void take(std::uint64_t iteration, const std::vector<std::uint8_t>& unique);
  const std::vector<std::uint8_t>* framed(std::uint64_t iteration) const;
  std::optional<std::uint64_t> newest() const;
  std::optional<std::uint64_t> previous() const;
  Role role() const { return role_; }
  std::uint64_t capacity() const { return capacity_; }
  // B200 extension (not in the reference API): the per-slice FNV-1a-64
  // table of the most recent take(), copied to host memory without framing
  // the payload; returns the number of entries copied (<= max).
  std::uint64_t last_slice_checksums(std::uint64_t* host, std::uint64_t max) const;

 private:
  Role role_;
  std::uint64_t capacity_;
  std::unique_ptr<detail::Slots> slots_;
};

class NeighborBuffer {
 public:
  explicit NeighborBuffer(Role origin);
  ~NeighborBuffer();
  NeighborBuffer(NeighborBuffer&&) noexcept;
  NeighborBuffer& operator=(NeighborBuffer&&) noexcept;

  void store(std::vector<std::uint8_t> framed);
  const std::vector<std::uint8_t>* framed_at(std::uint64_t iteration) const;
  std::optional<std::uint64_t> newest() const;
  Role origin() const { return origin_; }
  void clear();

 private:
  Role origin_;
  std::unique_ptr<detail::Slots> slots_;
};

struct RestorePieces {
  const std::vector<std::uint8_t>* unique = nullptr;
  const std::vector<std::uint8_t>* weights = nullptr;
  const std::vector<std::uint8_t>* optimizer = nullptr;
};

StateBundle assemble_restore(const Role& who, std::uint64_t target, const UniquenessPlan& plan,
                             const RestorePieces& pieces);
StateBundle restore_from_fallback(const store::Storage& storage, const Role& who,
                                  std::uint64_t iteration);

}  // namespace ftsim::ckpt
