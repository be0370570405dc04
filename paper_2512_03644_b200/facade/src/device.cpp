// device.cpp -- facade plumbing: device choice, error mapping, staging.
#include "device.hpp"

#include <cstdlib>
#include <stdexcept>

namespace ftsim::b200 {

int device() {
  static const int dev = [] {
    const char* e = std::getenv("FFX_DEVICE");
    return e ? std::atoi(e) : 0;
  }();
  return dev;
}

void raise(int status, const char* what) {
  std::string msg = std::string(what) + ": " + ffx_last_error();
  switch (status) {
    case FFX_ECONFIG: throw ckpt::ConfigError(msg);
    case FFX_EVERSION: throw ckpt::VersionError(msg);
    case FFX_ERESTORE: throw ckpt::RestoreError(msg);
    case FFX_ECORRUPT: throw store::CorruptSnapshot(msg);
    case FFX_EINVAL: throw std::invalid_argument(msg);
    case FFX_ERANGE: throw std::out_of_range(msg);
    case FFX_ENOMEM: throw std::bad_alloc();
    default: throw std::runtime_error(msg);
  }
}

void DevBuf::reset(std::uint64_t bytes) {
  release();
  check(ffx_device_alloc(device(), bytes, &p_), "device_alloc");
  n_ = bytes;
}

void DevBuf::release() {
  if (p_) ffx_device_free(device(), p_);
  p_ = nullptr;
  n_ = 0;
}

bool is_device_ptr(const void* p) {
  int d = 0;
  ffx_pointer_is_device(p, &d);
  return d != 0;
}

const std::uint8_t* on_device(const void* p, std::size_t len, DevBuf& scratch) {
  if (len == 0) return nullptr;
  if (is_device_ptr(p)) return static_cast<const std::uint8_t*>(p);
  scratch.ensure(len);
  check(ffx_memcpy(scratch.get(), p, len, nullptr, 1), "stage to device");
  return scratch.get();
}

std::uint64_t device_checksum(const void* p, std::size_t len) {
  static thread_local DevBuf scratch;
  std::uint64_t h = 0;
  const std::uint8_t* d = on_device(p, len, scratch);
  check(ffx_checksum64(d, len, &h, nullptr), "checksum64");
  return h;
}

}  // namespace ftsim::b200
