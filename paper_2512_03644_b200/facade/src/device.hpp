// device.hpp -- facade-internal plumbing over the C ABI (include/ffx.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <mutex>
#include <stdexcept>
#include <string>

#include "ffx.h"
#include "ftsim/ckpt.hpp"
#include "ftsim/storage.hpp"

namespace ftsim::b200 {

// The GPU the facade works on: $FFX_DEVICE, default 0.
int device();

// Status -> the reference's exception types (ckpt.hpp:58-68,
// storage.hpp:55-57, storage.cpp:49, domain.cpp:22).
[[noreturn]] void raise(int status, const char* what);
inline void check(int status, const char* what) {
  if (status != FFX_OK) raise(status, what);
}

// Owned device allocation.
class DevBuf {
 public:
  DevBuf() = default;
  explicit DevBuf(std::uint64_t bytes) { reset(bytes); }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  void reset(std::uint64_t bytes);
  void ensure(std::uint64_t bytes) { if (bytes > n_) reset(bytes); }
  void release();
  std::uint8_t* get() const { return static_cast<std::uint8_t*>(p_); }
  std::uint64_t size() const { return n_; }

 private:
  void* p_ = nullptr;
  std::uint64_t n_ = 0;
};

bool is_device_ptr(const void* p);

// A device view of caller bytes: the pointer itself when it is device
// memory, else a staged (H2D) copy in `scratch`.
const std::uint8_t* on_device(const void* p, std::size_t len, DevBuf& scratch);

// Device-resident FNV-1a-64 of caller bytes (host or device).
std::uint64_t device_checksum(const void* p, std::size_t len);

}  // namespace ftsim::b200
