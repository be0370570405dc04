// ckpt.cpp -- facade: razor, device-resident version slots, restore.
//
// HostSnapshots / NeighborBuffer keep the reference's observable contract
// (ckpt.cpp:35-105): fixed capacity and ConfigError, two retained versions,
// replace-in-place of a held iteration, validate-before-accept on the holder.
// The versions live in an ffx replica (two device slots, fused copy +
// per-slice FNV on the way in); SNP1 bytes are produced only when a caller
// asks for framed()/framed_at().
#include <algorithm>
#include <deque>
#include <map>
#include <string>

#include "device.hpp"
#include "ftsim/ckpt.hpp"
#include "ftsim/hash.hpp"

namespace ftsim::ckpt {

using store::BlobKind;

UniquenessPlan razor(const ClusterSpec& spec) {
  ffx_cluster_spec c{};
  c.num_nodes = spec.num_nodes;
  c.gpus_per_node = spec.gpus_per_node ? spec.gpus_per_node : 1;
  c.data_parallel = spec.data_parallel;
  c.pipeline_parallel = spec.pipeline_parallel ? spec.pipeline_parallel : 1;
  c.tensor_parallel = spec.tensor_parallel ? spec.tensor_parallel : 1;
  c.distributed_optimizer = spec.distributed_optimizer;
  c.params_per_device = spec.params_per_device;
  ffx_uniqueness_plan p{};
  b200::check(ffx_razor(&c, &p), "razor");
  return UniquenessPlan{p.weights_redundant != 0, p.optimizer_redundant != 0, p.unique_bytes_per_device};
}

LazyKinds lazy_kinds(const UniquenessPlan& plan) {
  return LazyKinds{plan.weights_redundant, plan.optimizer_redundant};
}

int version_for_target(std::uint64_t held, std::uint64_t target) {
  int v = 0;
  b200::check(ffx_version_for_target(held, target, &v), "version_for_target");
  return v;
}

namespace detail {

// Two device slots for one role plus the frames already exported from them.
struct Slots {
  Role role;
  ffx_ctx* ctx = nullptr;
  ffx_replica* rep = nullptr;
  std::uint64_t cap = 0;
  b200::DevBuf staging;
  std::deque<std::uint64_t> kept;  // oldest first, at most two
  struct Frame {
    bool fresh = false;
    std::vector<std::uint8_t> bytes;
  };
  mutable std::map<std::uint64_t, Frame> frames;

  explicit Slots(Role r) : role(r) {
    ffx_cluster_spec spec{1, 1, 1, 1, 1, 0, 1};
    b200::check(ffx_open(b200::device(), &spec, ffx_role{r.dp, r.pp, r.tp}, 0, &ctx), "open");
  }
  ~Slots() {
    if (rep) ffx_replica_destroy(rep);
    if (ctx) ffx_close(ctx);
  }

  void allocate(std::uint64_t capacity) {
    ffx_replica* fresh = nullptr;
    b200::check(ffx_replica_create(ctx, ffx_role{role.dp, role.pp, role.tp}, capacity, 2, &fresh),
                "replica_create");
    if (rep) ffx_replica_destroy(rep);
    rep = fresh;
    cap = capacity;
    b200::check(ffx_snapshot_target(ctx, rep), "snapshot_target");
  }

  // Snapshot `len` bytes as `iteration`: from device memory (dev; nullptr
  // when len == 0), or from host memory (host), copied into the staging
  // buffer under the snapshot's own batches (ffx_snapshot_from_host).
  void write(std::uint64_t iteration, const std::uint8_t* dev, std::uint64_t len, const void* host = nullptr) {
    if (host) {
      staging.ensure(len);
      dev = staging.get();
    } else if (len && reinterpret_cast<std::uintptr_t>(dev) % 16 != 0) {
      staging.ensure(len);  // the kernels want 16-byte aligned regions
      b200::check(ffx_memcpy(staging.get(), dev, len, nullptr, 1), "align copy");
      dev = staging.get();
    }
    b200::check(ffx_clear_regions(ctx), "clear_regions");
    b200::check(ffx_register_region(ctx, FFX_REGION_BLOB, const_cast<std::uint8_t*>(dev), len, 1),
                "register_region");
    if (host) {
      b200::check(ffx_snapshot_from_host(ctx, iteration, host, len, 0, nullptr), "snapshot_from_host");
    } else {
      ffx_snapshot_opts o{};
      b200::check(ffx_snapshot(ctx, iteration, nullptr, &o), "snapshot");
    }
    b200::check(ffx_stream_sync(nullptr), "sync");  // take()/store() complete on return
    if (auto f = frames.find(iteration); f != frames.end()) f->second.fresh = false;
    if (std::find(kept.begin(), kept.end(), iteration) == kept.end()) {
      kept.push_back(iteration);
      while (kept.size() > 2) {
        frames.erase(kept.front());
        kept.pop_front();
      }
    }
  }

  const std::vector<std::uint8_t>* frame(std::uint64_t iteration) const {
    if (std::find(kept.begin(), kept.end(), iteration) == kept.end()) return nullptr;
    Frame& f = frames[iteration];
    if (!f.fresh) {
      std::uint64_t n = 0;
      b200::check(ffx_replica_export_frame(rep, iteration, nullptr, 0, &n, nullptr), "export_frame");
      f.bytes.resize(n);
      b200::check(ffx_replica_export_frame(rep, iteration, f.bytes.data(), n, &n, nullptr), "export_frame");
      f.fresh = true;
    }
    return &f.bytes;
  }

  void clear() {
    if (rep) b200::check(ffx_replica_clear(rep), "replica_clear");
    kept.clear();
    frames.clear();
  }
};

}  // namespace detail

// ---- HostSnapshots -------------------------------------------------------------

HostSnapshots::HostSnapshots(Role role, std::uint64_t capacity_bytes)
    : role_(role), capacity_(capacity_bytes), slots_(std::make_unique<detail::Slots>(role)) {
  slots_->allocate(capacity_bytes);
}
HostSnapshots::~HostSnapshots() = default;
HostSnapshots::HostSnapshots(HostSnapshots&&) noexcept = default;
HostSnapshots& HostSnapshots::operator=(HostSnapshots&&) noexcept = default;

void HostSnapshots::take(std::uint64_t iteration, const void* unique, std::size_t len) {
  if (len > capacity_)
    throw ConfigError("snapshot payload " + std::to_string(len) + " exceeds the host buffer of " +
                      std::to_string(capacity_) + " bytes");
  if (len && !b200::is_device_ptr(unique)) {  // host memory: copied in under the snapshot
    slots_->write(iteration, nullptr, len, unique);
    return;
  }
  slots_->write(iteration, static_cast<const std::uint8_t*>(unique), len);
}

void HostSnapshots::take(std::uint64_t iteration, const std::vector<std::uint8_t>& unique) {
  take(iteration, unique.data(), unique.size());
}

const std::vector<std::uint8_t>* HostSnapshots::framed(std::uint64_t iteration) const {
  return slots_->frame(iteration);
}

std::uint64_t HostSnapshots::last_slice_checksums(std::uint64_t* host, std::uint64_t max) const {
  std::uint64_t n = 0;
  b200::check(ffx_snapshot_read_sums(slots_->ctx, host, max, &n, nullptr), "read_sums");
  b200::check(ffx_stream_sync(nullptr), "sync");
  return n;
}

std::optional<std::uint64_t> HostSnapshots::newest() const {
  if (slots_->kept.empty()) return std::nullopt;
  return slots_->kept.back();
}

std::optional<std::uint64_t> HostSnapshots::previous() const {
  if (slots_->kept.size() < 2) return std::nullopt;
  return slots_->kept[slots_->kept.size() - 2];
}

// ---- NeighborBuffer ------------------------------------------------------------

NeighborBuffer::NeighborBuffer(Role origin)
    : origin_(origin), slots_(std::make_unique<detail::Slots>(origin)) {}
NeighborBuffer::~NeighborBuffer() = default;
NeighborBuffer::NeighborBuffer(NeighborBuffer&&) noexcept = default;
NeighborBuffer& NeighborBuffer::operator=(NeighborBuffer&&) noexcept = default;

void NeighborBuffer::store(std::vector<std::uint8_t> framed) {
  // Validate exactly as unpack_blob does (storage.cpp:92-101), with the
  // checksum computed on the device over the staged payload, which is then
  // the snapshot source -- one H2D for verify + store.
  const store::BlobInfo info = store::parse_header(framed.data(), framed.size());
  if (framed.size() != store::kHeaderBytes + info.payload_len)
    throw store::CorruptSnapshot("snapshot length disagrees with header");
  const std::uint8_t* dev =
      b200::on_device(framed.data() + store::kHeaderBytes, info.payload_len, slots_->staging);
  std::uint64_t sum = 0;
  b200::check(ffx_checksum64(dev, info.payload_len, &sum, nullptr), "checksum64");
  if (sum != info.checksum) throw store::CorruptSnapshot("snapshot checksum mismatch");
  if (info.role != origin_)
    throw store::CorruptSnapshot("snapshot from " + info.role.str() + " offered to the buffer for " +
                                 origin_.str());
  if (info.kind != BlobKind::Optimizer)
    throw store::CorruptSnapshot("ring stream carries optimizer state only");

  if (!slots_->rep || info.payload_len > slots_->cap) {
    // Grow: carry the retained frames over into a larger replica.
    std::vector<std::pair<std::uint64_t, std::vector<std::uint8_t>>> carry;
    for (const std::uint64_t it : slots_->kept)
      if (it != info.iteration) carry.emplace_back(it, *slots_->frame(it));
    slots_->allocate(std::max<std::uint64_t>(info.payload_len, 2 * slots_->cap));
    slots_->kept.clear();
    slots_->frames.clear();
    b200::DevBuf tmp;
    for (auto& [it, f] : carry) {
      const std::uint64_t n = f.size() - store::kHeaderBytes;
      const std::uint8_t* d = b200::on_device(f.data() + store::kHeaderBytes, n, tmp);
      slots_->write(it, d, n);
    }
    if (!carry.empty())  // re-stage: `tmp` reuse may not have touched staging, but be explicit
      dev = b200::on_device(framed.data() + store::kHeaderBytes, info.payload_len, slots_->staging);
  }
  slots_->write(info.iteration, dev, info.payload_len);
}

const std::vector<std::uint8_t>* NeighborBuffer::framed_at(std::uint64_t iteration) const {
  return slots_->frame(iteration);
}

std::optional<std::uint64_t> NeighborBuffer::newest() const {
  if (slots_->kept.empty()) return std::nullopt;
  return slots_->kept.back();
}

void NeighborBuffer::clear() { slots_->clear(); }

// ---- restore ---------------------------------------------------------------------

namespace {

// ckpt.cpp:111-136 semantics: missing, invalid, wrong kind, stale, wrong role.
store::UnpackedBlob checked(const std::vector<std::uint8_t>* piece, const char* what, const Role& who,
                            std::uint64_t target, BlobKind kind, bool match_dp) {
  if (!piece) throw RestoreError(std::string(what) + " source missing");
  store::UnpackedBlob u;
  try {
    u = store::unpack_blob(*piece);
  } catch (const store::CorruptSnapshot& e) {
    throw RestoreError(std::string(what) + " source invalid: " + e.what());
  }
  if (u.info.kind != kind) throw RestoreError(std::string(what) + " source has the wrong kind");
  if (u.info.iteration != target)
    throw RestoreError(std::string(what) + " source is at iteration " + std::to_string(u.info.iteration) +
                       ", want " + std::to_string(target));
  const bool same = match_dp ? u.info.role == who : (u.info.role.pp == who.pp && u.info.role.tp == who.tp);
  if (!same) throw RestoreError(std::string(what) + " source is for " + u.info.role.str() + ", want " + who.str());
  return u;
}

}  // namespace

StateBundle assemble_restore(const Role& who, std::uint64_t target, const UniquenessPlan& plan,
                             const RestorePieces& pieces) {
  if (!plan.weights_redundant)
    throw RestoreError("no replica holds this state; only the full checkpoint path applies");
  StateBundle out;
  out.iteration = target;
  out.weights = checked(pieces.weights, "weights", who, target, BlobKind::Weights, false).payload;
  auto opt = plan.optimizer_redundant
                 ? checked(pieces.optimizer, "optimizer", who, target, BlobKind::Optimizer, false)
                 : checked(pieces.unique, "unique-state", who, target, BlobKind::Optimizer, true);
  out.optimizer_current = VersionedBlob{target, std::move(opt.payload)};
  out.optimizer_previous = VersionedBlob{target, {}};
  return out;
}

StateBundle restore_from_fallback(const store::Storage& storage, const Role& who, std::uint64_t iteration) {
  auto w = storage.get(who, iteration, BlobKind::Weights);
  auto o = storage.get(who, iteration, BlobKind::Optimizer);
  if (!w || !o)
    throw RestoreError("full checkpoint for " + who.str() + " at " + std::to_string(iteration) +
                       " is missing or invalid");
  StateBundle out;
  out.iteration = iteration;
  out.weights = std::move(*w);
  out.optimizer_current = VersionedBlob{iteration, std::move(*o)};
  out.optimizer_previous = VersionedBlob{iteration, {}};
  return out;
}

}  // namespace ftsim::ckpt
