/* ftsim_capi.h -- C entry points to the C++ facade (libftsim_b200.so) for
 * hosts that cannot link C++: ctypes (bench.py's end-to-end leg), cgo, JNI.
 *
 * The reference interface is a C++ class, ckpt::HostSnapshots
 * (proj/include/ftsim/ckpt.hpp:82-101, proj/src/ckpt.cpp:35-75); these wrap
 * the facade's drop-in implementation of it (facade/src/ckpt.cpp) one call per
 * method.  Status codes are ffx_status (include/ffx.h): the reference's
 * exceptions map 1:1 (ConfigError -> FFX_ECONFIG, RestoreError ->
 * FFX_ERESTORE, CorruptSnapshot -> FFX_ECORRUPT, invalid_argument ->
 * FFX_EINVAL, out_of_range -> FFX_ERANGE); ftsim_last_error() keeps the
 * message of the calling thread's last failure. */
#ifndef FTSIM_CAPI_H
#define FTSIM_CAPI_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* ftsim_last_error(void);
/* HostSnapshots(Role{dp, pp, tp}, capacity)                 ckpt.hpp:84 */
int ftsim_hs_create(uint16_t dp, uint16_t pp, uint16_t tp, uint64_t capacity, void** out);
int ftsim_hs_destroy(void* hs);
/* take(iteration, ptr, len): ptr in host or device memory    ckpt.cpp:38-53 */
int ftsim_hs_take(void* hs, uint64_t iteration, const void* data, uint64_t len);
/* newest() (FFX_ERESTORE when empty)                         ckpt.cpp:67-71 */
int ftsim_hs_newest(void* hs, uint64_t* iteration);
/* framed(iteration) copied out; dst NULL = size query         ckpt.cpp:60-66 */
int ftsim_hs_framed(void* hs, uint64_t iteration, void* dst, uint64_t cap, uint64_t* len);
/* B200 extension: the last take()'s per-slice FNV-1a-64 table (no framing). */
int ftsim_hs_last_sums(void* hs, uint64_t* host, uint64_t max, uint64_t* n);

#ifdef __cplusplus
}
#endif

#endif /* FTSIM_CAPI_H */
