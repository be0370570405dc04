// ftsim/evolution.hpp -- B200 facade: deterministic synthetic training state.
//
// Drop-in for proj/include/ftsim/evolution.hpp.  Digest recurrences stay on
// the host (32-byte SHA-256 keys); blob expansion and soundness checks --
// the bulk byte work -- run in the sm_100a kernels (ffx_expand,
// ffx_materialize, ffx_blob_check).
#pragma once

#include <cstdint>
#include <vector>

#include "ftsim/domain.hpp"
#include "ftsim/hash.hpp"

namespace ftsim::evo {

constexpr std::size_t kGradLanes = 8;

std::uint64_t weights_bytes(const ClusterSpec& spec);    // 2 B/param
std::uint64_t optimizer_bytes(const ClusterSpec& spec);  // 12 B/param, sharded over d

Digest weights_init(std::uint64_t seed, const Role& r);
Digest optimizer_init(std::uint64_t seed, const Role& r, bool distributed);
Digest weights_next(const Digest& w, const Digest& grad);
Digest optimizer_next(const Digest& o, const Digest& grad);
std::vector<std::uint64_t> grad_contribution(std::uint64_t seed, const Role& r,
                                             std::uint64_t iteration, std::uint64_t data_fold);
Digest grad_digest(const std::vector<std::uint64_t>& lanes);

std::vector<std::uint8_t> expand(const Digest& d, std::uint64_t bytes);
std::vector<std::uint8_t> materialize(const Digest& d, std::uint64_t bytes);
Digest digest_of_blob(const std::vector<std::uint8_t>& blob);
bool blob_is_sound(const std::vector<std::uint8_t>& blob);

Digest data_item_digest(std::uint64_t data_seed, std::uint64_t index);
std::vector<std::uint8_t> data_item(std::uint64_t data_seed, std::uint64_t index,
                                    std::uint32_t item_bytes);
std::uint64_t item_fold(const std::vector<std::uint8_t>& item);

std::uint64_t mix64(std::uint64_t x);

}  // namespace ftsim::evo
