// capi.cpp -- a C entry point to the facade's HostSnapshots for callers that
// cannot link C++ (ctypes: bench.py's end-to-end leg, a cgo/JNI host).  The
// reference-facing call is HostSnapshots::take(it, ptr, len) (ckpt.cpp:38-53,
// facade/src/ckpt.cpp); exceptions become the ffx status codes they map from
// (device.cpp raise()), the message is kept for ftsim_last_error().
#include <cstdint>
#include <exception>
#include <new>
#include <stdexcept>
#include <string>

#include "device.hpp"
#include "ftsim_capi.h"
#include "ftsim/ckpt.hpp"
#include "ftsim/storage.hpp"

namespace {

thread_local std::string g_msg;

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return FFX_OK;
  } catch (const ftsim::ckpt::ConfigError& e) {
    g_msg = e.what();
    return FFX_ECONFIG;
  } catch (const ftsim::ckpt::VersionError& e) {
    g_msg = e.what();
    return FFX_EVERSION;
  } catch (const ftsim::ckpt::RestoreError& e) {
    g_msg = e.what();
    return FFX_ERESTORE;
  } catch (const ftsim::store::CorruptSnapshot& e) {
    g_msg = e.what();
    return FFX_ECORRUPT;
  } catch (const std::invalid_argument& e) {
    g_msg = e.what();
    return FFX_EINVAL;
  } catch (const std::out_of_range& e) {
    g_msg = e.what();
    return FFX_ERANGE;
  } catch (const std::bad_alloc&) {
    g_msg = "out of memory";
    return FFX_ENOMEM;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return FFX_ECUDA;
  }
}

}  // namespace

extern "C" {

const char* ftsim_last_error(void) { return g_msg.c_str(); }

int ftsim_hs_create(uint16_t dp, uint16_t pp, uint16_t tp, uint64_t capacity, void** out) {
  if (!out) return FFX_EINVAL;
  return guarded([&] { *out = new ftsim::ckpt::HostSnapshots(ftsim::Role{dp, pp, tp}, capacity); });
}

int ftsim_hs_destroy(void* h) {
  return guarded([&] { delete static_cast<ftsim::ckpt::HostSnapshots*>(h); });
}

/* HostSnapshots::take(iteration, ptr, len): ptr may be host or device memory. */
int ftsim_hs_take(void* h, uint64_t iteration, const void* data, uint64_t len) {
  if (!h) return FFX_EINVAL;
  return guarded([&] { static_cast<ftsim::ckpt::HostSnapshots*>(h)->take(iteration, data, len); });
}

/* newest(): FFX_ERESTORE when nothing is held. */
int ftsim_hs_newest(void* h, uint64_t* iteration) {
  if (!h || !iteration) return FFX_EINVAL;
  return guarded([&] {
    const auto n = static_cast<ftsim::ckpt::HostSnapshots*>(h)->newest();
    if (!n) throw ftsim::ckpt::RestoreError("no snapshot held");
    *iteration = *n;
  });
}

/* The last take()'s per-slice checksum table into host memory. */
int ftsim_hs_last_sums(void* h, uint64_t* host, uint64_t max, uint64_t* n) {
  if (!h || !n) return FFX_EINVAL;
  return guarded([&] { *n = static_cast<ftsim::ckpt::HostSnapshots*>(h)->last_slice_checksums(host, max); });
}

/* framed(iteration) copied out (SNP1 bytes; *len = 32 + payload).  dst NULL:
 * size query. */
int ftsim_hs_framed(void* h, uint64_t iteration, void* dst, uint64_t cap, uint64_t* len) {
  if (!h || !len) return FFX_EINVAL;
  return guarded([&] {
    const auto* f = static_cast<ftsim::ckpt::HostSnapshots*>(h)->framed(iteration);
    if (!f) throw ftsim::ckpt::RestoreError("iteration not held");
    *len = f->size();
    if (dst) {
      if (cap < f->size()) throw ftsim::ckpt::ConfigError("destination too small");
      std::copy(f->begin(), f->end(), static_cast<std::uint8_t*>(dst));
    }
  });
}

}  // extern "C"
