// hash_domain.cpp -- facade: digests, checksum64, role layout.
//
// SHA-256 uses OpenSSL EVP exactly as the reference does (hash.cpp:19-33,
// HashIn :52-100): it only ever sees 32-byte keys.  checksum64 runs on the
// GPU.  Layout functions call the C ABI (domain.cpp:18-62 restated there).
#include <openssl/evp.h>

#include <stdexcept>

#include "device.hpp"
#include "ftsim/domain.hpp"
#include "ftsim/hash.hpp"

namespace ftsim {

namespace {

void ok(int rc, const char* what) {
  if (rc != 1) throw std::runtime_error(std::string("digest failure in ") + what);
}

ffx_cluster_spec to_c(const ClusterSpec& s) {
  ffx_cluster_spec c{};
  c.num_nodes = s.num_nodes;
  c.gpus_per_node = s.gpus_per_node;
  c.data_parallel = s.data_parallel;
  c.pipeline_parallel = s.pipeline_parallel;
  c.tensor_parallel = s.tensor_parallel;
  c.distributed_optimizer = s.distributed_optimizer ? 1u : 0u;
  c.params_per_device = s.params_per_device;
  return c;
}

ffx_role to_c(const Role& r) { return ffx_role{r.dp, r.pp, r.tp}; }
Role from_c(const ffx_role& r) { return Role{r.dp, r.pp, r.tp}; }

}  // namespace

// ---- hash --------------------------------------------------------------------

Digest sha256(const void* data, std::size_t len) {
  Digest out{};
  unsigned int n = 0;
  ok(EVP_Digest(data, len, out.data(), &n, EVP_sha256(), nullptr), "EVP_Digest");
  return out;
}
Digest sha256(const std::vector<std::uint8_t>& data) { return sha256(data.data(), data.size()); }
Digest sha256(const std::string& data) { return sha256(data.data(), data.size()); }

std::string hex(const Digest& d) {
  static const char digits[] = "0123456789abcdef";
  std::string s(64, '0');
  for (std::size_t i = 0; i < d.size(); ++i) {
    s[2 * i] = digits[d[i] >> 4];
    s[2 * i + 1] = digits[d[i] & 15];
  }
  return s;
}

std::uint64_t fold64(const Digest& d) {
  std::uint64_t v = 0;
  for (int i = 0; i < 8; ++i) v |= static_cast<std::uint64_t>(d[i]) << (8 * i);
  return v;
}

HashIn::HashIn() : ctx_(EVP_MD_CTX_new()) {
  if (!ctx_) throw std::runtime_error("EVP_MD_CTX_new failed");
  ok(EVP_DigestInit_ex(static_cast<EVP_MD_CTX*>(ctx_), EVP_sha256(), nullptr), "DigestInit");
}
HashIn::~HashIn() { EVP_MD_CTX_free(static_cast<EVP_MD_CTX*>(ctx_)); }

HashIn& HashIn::bytes(const void* data, std::size_t len) {
  ok(EVP_DigestUpdate(static_cast<EVP_MD_CTX*>(ctx_), data, len), "DigestUpdate");
  return *this;
}
HashIn& HashIn::u64(std::uint64_t v) {
  std::uint8_t b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<std::uint8_t>(v >> (8 * i));
  return bytes(b, 8);
}
HashIn& HashIn::u32(std::uint32_t v) {
  std::uint8_t b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<std::uint8_t>(v >> (8 * i));
  return bytes(b, 4);
}
HashIn& HashIn::u16(std::uint16_t v) {
  const std::uint8_t b[2] = {static_cast<std::uint8_t>(v), static_cast<std::uint8_t>(v >> 8)};
  return bytes(b, 2);
}
HashIn& HashIn::u8(std::uint8_t v) { return bytes(&v, 1); }
HashIn& HashIn::str(const std::string& s) { return u64(s.size()).bytes(s.data(), s.size()); }
Digest HashIn::digest() {
  Digest out{};
  unsigned int n = 0;
  ok(EVP_DigestFinal_ex(static_cast<EVP_MD_CTX*>(ctx_), out.data(), &n), "DigestFinal");
  return out;
}

std::uint64_t checksum64(const void* data, std::size_t len) { return b200::device_checksum(data, len); }
std::uint64_t checksum64(const std::vector<std::uint8_t>& data) {
  return checksum64(data.data(), data.size());
}

// ---- domain --------------------------------------------------------------------

std::string Role::str() const {
  return "d" + std::to_string(dp) + "p" + std::to_string(pp) + "t" + std::to_string(tp);
}
std::string TID::str() const { return role.str() + "@" + std::to_string(iteration); }

Role role_of(std::uint32_t global_index, const ClusterSpec& spec) {
  const auto c = to_c(spec);
  ffx_role r{};
  b200::check(ffx_role_of(&c, global_index, &r), "role_of");
  return from_c(r);
}

std::uint32_t index_of(const Role& role, const ClusterSpec& spec) {
  const auto c = to_c(spec);
  std::uint32_t i = 0;
  b200::check(ffx_index_of(&c, to_c(role), &i), "index_of");
  return i;
}

WorkerId placement_of(const Role& role, const ClusterSpec& spec) {
  const std::uint32_t i = index_of(role, spec);
  return WorkerId{i / spec.gpus_per_node, static_cast<std::uint16_t>(i % spec.gpus_per_node)};
}

std::uint32_t node_of(const Role& role, const ClusterSpec& spec) {
  const auto c = to_c(spec);
  std::uint32_t n = 0;
  b200::check(ffx_node_of(&c, to_c(role), &n), "node_of");
  return n;
}

Role dp_neighbor(const Role& role, const ClusterSpec& spec) {
  const auto c = to_c(spec);
  ffx_role r{};
  b200::check(ffx_dp_neighbor(&c, to_c(role), &r), "dp_neighbor");
  return from_c(r);
}

Role dp_predecessor(const Role& role, const ClusterSpec& spec) {
  const auto c = to_c(spec);
  ffx_role r{};
  b200::check(ffx_dp_predecessor(&c, to_c(role), &r), "dp_predecessor");
  return from_c(r);
}

std::vector<std::string> validate_spec(const ClusterSpec& s) {
  std::vector<std::string> errs;
  const auto need = [&errs](bool cond, std::string msg) {
    if (!cond) errs.push_back(std::move(msg));
  };
  need(s.num_nodes != 0, "num_nodes must be nonzero");
  need(s.gpus_per_node != 0, "gpus_per_node must be nonzero");
  need(s.data_parallel != 0, "data_parallel must be nonzero");
  need(s.pipeline_parallel != 0, "pipeline_parallel must be nonzero");
  need(s.tensor_parallel != 0, "tensor_parallel must be nonzero");
  need(s.seq_len != 0, "seq_len must be nonzero");
  need(s.batch_size != 0, "batch_size must be nonzero");
  need(s.params_per_device != 0, "params_per_device must be nonzero");
  need(s.preload_depth != 0, "preload_depth must be nonzero");
  need(s.gpu_mtbf_hours > 0.0, "gpu_mtbf_hours must be positive");
  need(s.nic_bw > 0.0, "nic_bw must be positive");
  need(s.disk_bw > 0.0, "disk_bw must be positive");
  need(s.compute_flops > 0.0, "compute_flops must be positive");
  need(s.ckpt_interval_hours > 0.0, "ckpt_interval_hours must be positive");
  const std::uint64_t degrees =
      std::uint64_t{s.data_parallel} * s.pipeline_parallel * s.tensor_parallel;
  const std::uint64_t world = std::uint64_t{s.num_nodes} * s.gpus_per_node;
  if (s.num_nodes && s.gpus_per_node && degrees != world)
    errs.push_back("data_parallel * pipeline_parallel * tensor_parallel (" + std::to_string(degrees) +
                   ") must equal num_nodes * gpus_per_node (" + std::to_string(world) + ")");
  if (s.tensor_parallel && s.gpus_per_node && s.tensor_parallel > s.gpus_per_node)
    errs.push_back("tensor_parallel must not exceed gpus_per_node");
  return errs;
}

}  // namespace ftsim
