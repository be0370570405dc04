/*
 * ffx_oracle.c -- CPU restatement of FFTrainer's state-backup arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * path; it is imported by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg, never by the product library (libffx.so) and never on a
 * measured path.  Each function cites the reference line it restates
 * (paths relative to the reference checkout's proj/ directory).
 *
 * Parity pin: tests/test_oracle.py checks every function below against
 *   (a) the reference's own known-answer tests (proj/tests/test_evolution.cpp:44-50,
 *       proj/tests/test_ckpt.cpp:50-72), and
 *   (b) fixtures in tests/golden/ produced by the reference itself
 *       (oracle/_ref/libftsim_ref.so, compiled from proj/src by oracle/Makefile,
 *       fixtures written by oracle/gen_golden.py).
 *
 * All arithmetic is integer, little-endian, mod 2^64.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>

#include <openssl/evp.h>

#define ORC_FNV_BASIS 0xcbf29ce484222325ull /* hash.cpp:104 */
#define ORC_FNV_PRIME 0x100000001b3ull      /* hash.cpp:107 */
#define ORC_GOLDEN 0x9E3779B97F4A7C15ull    /* evolution.cpp:44, :76 */

/* hash.cpp:102-110 -- FNV-1a 64, byte serial. */
uint64_t orc_fnv1a64(const uint8_t* p, uint64_t n) {
  uint64_t h = ORC_FNV_BASIS;
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= ORC_FNV_PRIME;
  }
  return h;
}

/* FNV-1a continued from an arbitrary state (used to build slice/segment
 * checks; with h = ORC_FNV_BASIS it is exactly hash.cpp:102-110). */
uint64_t orc_fnv1a64_from(uint64_t h, const uint8_t* p, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= ORC_FNV_PRIME;
  }
  return h;
}

/* Per-slice checksum table: out[s] = checksum64(p[s*slice, min((s+1)*slice, n))).
 * The B200 format's integrity unit; each entry is the reference function
 * hash.cpp:102-110 applied verbatim to one contiguous slice. */
uint64_t orc_slice_fnv(const uint8_t* p, uint64_t n, uint64_t slice, uint64_t* out) {
  if (slice == 0) return 0;
  uint64_t ns = (n + slice - 1) / slice;
  for (uint64_t s = 0; s < ns; ++s) {
    uint64_t off = s * slice;
    uint64_t len = (n - off) < slice ? (n - off) : slice;
    out[s] = orc_fnv1a64(p + off, len);
  }
  return ns;
}

/* hash.cpp:46-50 -- first eight digest bytes, little-endian. */
uint64_t orc_fold64(const uint8_t* d) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | d[i];
  return v;
}

/* evolution.cpp:43-48 -- note the leading golden-ratio add. */
uint64_t orc_mix64(uint64_t x) {
  x += ORC_GOLDEN;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* evolution.cpp:71-86 -- word k (0-based) is mix64(fold64(d) + (k+1)*G),
 * stored little-endian; a trailing partial word is truncated. */
void orc_expand(const uint8_t* d, uint64_t bytes, uint8_t* out) {
  uint64_t s = orc_fold64(d);
  uint64_t i = 0;
  while (i < bytes) {
    s += ORC_GOLDEN;
    uint64_t v = orc_mix64(s);
    for (int b = 0; b < 8 && i < bytes; ++b) out[i++] = (uint8_t)(v >> (8 * b));
  }
}

/* evolution.cpp:88-97 -- digest prefix then expansion.  Returns -1 where the
 * reference throws std::invalid_argument (bytes < 32). */
int orc_materialize(const uint8_t* d, uint64_t bytes, uint8_t* out) {
  if (bytes < 32) return -1;
  memcpy(out, d, 32);
  orc_expand(d, bytes - 32, out + 32);
  return 0;
}

/* evolution.cpp:106-110 -- 1 when blob == materialize(prefix, size). */
int orc_blob_is_sound(const uint8_t* blob, uint64_t n) {
  if (n < 32) return 0;
  uint64_t s = orc_fold64(blob);
  uint64_t i = 32;
  while (i < n) {
    s += ORC_GOLDEN;
    uint64_t v = orc_mix64(s);
    for (int b = 0; b < 8 && i < n; ++b, ++i)
      if (blob[i] != (uint8_t)(v >> (8 * b))) return 0;
  }
  return 1;
}

/* evolution.cpp:11-19 */
uint64_t orc_weights_bytes(uint64_t phi) { return 2 * phi; }
uint64_t orc_optimizer_bytes(uint64_t phi, uint32_t d, int distributed) {
  uint64_t full = 12 * phi;
  if (!distributed || d <= 1) return full;
  return (full + d - 1) / d;
}

/* ckpt.cpp:13-21 -- out[0]=weights_redundant, out[1]=optimizer_redundant,
 * return = unique bytes per device. */
uint64_t orc_razor(uint64_t phi, uint32_t d, int distributed, int* flags) {
  int wr = d > 1;
  int orr = d > 1 && !distributed;
  flags[0] = wr;
  flags[1] = orr;
  return orr ? 0 : orc_optimizer_bytes(phi, d, distributed);
}

/* ckpt.cpp:27-33 -- 0 current, 1 previous, -1 where the reference throws
 * VersionError. */
int orc_version_for_target(uint64_t held, uint64_t target) {
  if (held == target) return 0;
  if (held == target + 1) return 1;
  return -1;
}

static void le16(uint8_t* p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void le32(uint8_t* p, uint32_t v) { for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i)); }
static void le64(uint8_t* p, uint64_t v) { for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i)); }
static uint64_t rd(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

/* storage.cpp:45-66 -- the 32-byte SNP1 header (layout storage.hpp:12-25).
 * Returns -1 where the reference throws (payload over the u32 length). */
int orc_pack_header(uint16_t dp, uint16_t pp, uint16_t tp, uint64_t iteration,
                    uint8_t kind, uint64_t len, uint64_t checksum, uint8_t* h) {
  if (len > 0xffffffffull) return -1;
  memset(h, 0, 32);
  le32(h + 0, 0x31504E53u); /* "SNP1" */
  h[4] = 1;                 /* kFormatVersion */
  h[5] = kind;
  le16(h + 6, dp);
  le16(h + 8, pp);
  le16(h + 10, tp);
  le64(h + 12, iteration);
  le32(h + 20, (uint32_t)len);
  le64(h + 24, checksum);
  return 0;
}

/* storage.cpp:45-66 -- full frame: header + payload. */
int orc_pack_blob(uint16_t dp, uint16_t pp, uint16_t tp, uint64_t iteration,
                  uint8_t kind, const uint8_t* payload, uint64_t len, uint8_t* out) {
  if (orc_pack_header(dp, pp, tp, iteration, kind, len, orc_fnv1a64(payload, len), out))
    return -1;
  if (len) memcpy(out + 32, payload, len);
  return 0;
}

/* storage.cpp:74-90 and :92-101.  fields: dp,pp,tp,iteration,kind,len,checksum.
 * Returns 0 ok, or a negative code naming the reference's CorruptSnapshot
 * branch: -1 short, -2 magic, -3 version, -4 kind, -5 length, -6 checksum. */
int orc_unpack(const uint8_t* f, uint64_t n, uint64_t* fields) {
  if (n < 32) return -1;
  if (rd(f, 4) != 0x31504E53u) return -2;
  if (f[4] != 1) return -3;
  if (f[5] > 1) return -4;
  fields[0] = rd(f + 6, 2);
  fields[1] = rd(f + 8, 2);
  fields[2] = rd(f + 10, 2);
  fields[3] = rd(f + 12, 8);
  fields[4] = f[5];
  fields[5] = rd(f + 20, 4);
  fields[6] = rd(f + 24, 8);
  if (n != 32 + fields[5]) return -5;
  if (orc_fnv1a64(f + 32, fields[5]) != fields[6]) return -6;
  return 0;
}

/* hash.cpp:19-33 via OpenSSL (the reference's own third-party SHA-256). */
int orc_sha256(const uint8_t* data, uint64_t len, uint8_t* out32) {
  unsigned int n = 0;
  return EVP_Digest(data, (size_t)len, out32, &n, EVP_sha256(), NULL) == 1 ? 0 : -1;
}

/* HashIn key layouts (hash.cpp:52-100): str = u64 length + bytes, ints LE. */
static size_t put_str(uint8_t* b, const char* s) {
  size_t n = strlen(s);
  le64(b, n);
  memcpy(b + 8, s, n);
  return 8 + n;
}

/* evolution.cpp:21-24 */
void orc_weights_init(uint64_t seed, uint16_t pp, uint16_t tp, uint8_t* out) {
  uint8_t b[64];
  size_t o = put_str(b, "W0");
  le64(b + o, seed); o += 8;
  le16(b + o, pp); o += 2;
  le16(b + o, tp); o += 2;
  orc_sha256(b, o, out);
}

/* evolution.cpp:26-31 */
void orc_optimizer_init(uint64_t seed, uint16_t dp, uint16_t pp, uint16_t tp,
                        int distributed, uint8_t* out) {
  uint8_t b[64];
  size_t o = put_str(b, "O0");
  le64(b + o, seed); o += 8;
  if (distributed) { le16(b + o, dp); o += 2; }
  le16(b + o, pp); o += 2;
  le16(b + o, tp); o += 2;
  orc_sha256(b, o, out);
}

/* evolution.cpp:33-41 -- tag "W" or "O", then state digest, then grad digest. */
void orc_state_next(const char* tag, const uint8_t* state, const uint8_t* grad, uint8_t* out) {
  uint8_t b[96];
  size_t o = put_str(b, tag);
  memcpy(b + o, state, 32); o += 32;
  memcpy(b + o, grad, 32); o += 32;
  orc_sha256(b, o, out);
}

/* ---- per-iteration state evolution (SURVEY 8(d) synthetic inputs) --------
 * The optimizer digest of a rank at iteration n:
 *   d_0 = optimizer_init(seed, role)                       evolution.cpp:26-31
 *   d_n = optimizer_next(d_{n-1}, grad_digest(grad_contribution(seed, role, n,
 *           window_fold(seed, window_of(assign, column, n)))))
 * optimizer_next :38-41, grad_contribution :50-62, grad_digest :64-69,
 * data_item_digest / data_item / item_fold :112-128 (8-byte items),
 * window_of dataloader.cpp:36-49, window_fold :166-171, the assignment
 * controller.cpp:127-140 (start 0: per_column = batch/world, base 0);
 * column = the rank's global index (domain.cpp:18-30). */

/* item_fold(data_item(seed, index, 8)) = the first expand() word of the item digest */
uint64_t orc_item_fold(uint64_t data_seed, uint64_t index) {
  uint8_t b[32], d[32];
  size_t o = put_str(b, "D");
  le64(b + o, data_seed); o += 8;
  le64(b + o, index); o += 8;
  orc_sha256(b, o, d);
  return orc_mix64(orc_fold64(d) + ORC_GOLDEN);
}

uint64_t orc_window_fold(uint64_t seed, uint64_t first, uint32_t count) {
  uint64_t acc = 0;
  for (uint32_t i = 0; i < count; ++i) acc += orc_item_fold(seed, first + i);
  return acc;
}

void orc_grad_contribution(uint64_t seed, uint16_t dp, uint16_t pp, uint16_t tp, uint64_t iteration,
                           uint64_t data_fold, uint64_t lanes[8]) {
  uint8_t b[64], d[32];
  size_t o = put_str(b, "C");
  le64(b + o, seed); o += 8;
  le16(b + o, dp); o += 2;
  le16(b + o, pp); o += 2;
  le16(b + o, tp); o += 2;
  le64(b + o, iteration); o += 8;
  orc_sha256(b, o, d);
  const uint64_t base = orc_fold64(d);
  for (int j = 0; j < 8; ++j) {
    const uint64_t off = (uint64_t)j * ORC_GOLDEN;
    lanes[j] = orc_mix64(base + off) + orc_mix64(data_fold + off);
  }
}

void orc_grad_digest(const uint64_t lanes[8], uint8_t* out) {
  uint8_t b[80];
  size_t o = put_str(b, "G");
  for (int j = 0; j < 8; ++j) { le64(b + o, lanes[j]); o += 8; }
  orc_sha256(b, o, out);
}

/* d_n for rank (dp,pp,tp) of a d x p x t grid with `batch` samples. */
int orc_optimizer_at(uint64_t seed, uint16_t dp, uint16_t pp, uint16_t tp, uint32_t d, uint32_t p,
                     uint32_t t, uint32_t batch, uint64_t n, int distributed, uint8_t* out) {
  const uint32_t world = d * p * t;
  if (world == 0 || batch % world != 0) return -1;  /* controller.cpp:131-132 SetupError */
  const uint32_t per_column = batch / world;
  const uint32_t column = ((uint32_t)dp * p + pp) * t + tp;
  uint8_t dig[32], g[32];
  uint64_t lanes[8];
  orc_optimizer_init(seed, dp, pp, tp, distributed, dig);
  for (uint64_t it = 1; it <= n; ++it) {
    const uint64_t first = it * (uint64_t)world * per_column + (uint64_t)column * per_column;
    orc_grad_contribution(seed, dp, pp, tp, it, orc_window_fold(seed, first, per_column), lanes);
    orc_grad_digest(lanes, g);
    orc_state_next("O", dig, g, dig);
  }
  memcpy(out, dig, 32);
  return 0;
}

/* Bytes [lo, lo+len) of materialize(d, total) without building the whole
 * blob (evolution.cpp:88-97 is counter-based: byte i >= 32 is byte (i-32)%8
 * of word (i-32)/8 of the expansion).  For spot checks of GB-sized state. */
int orc_materialize_range(const uint8_t* d, uint64_t total, uint64_t lo, uint64_t len, uint8_t* out) {
  if (total < 32 || lo + len > total) return -1;
  uint64_t s = orc_fold64(d);
  for (uint64_t k = 0; k < len; ++k) {
    uint64_t i = lo + k;
    if (i < 32) { out[k] = d[i]; continue; }
    uint64_t w = (i - 32) / 8;
    uint64_t v = orc_mix64(s + (w + 1) * ORC_GOLDEN);
    out[k] = (uint8_t)(v >> (8 * ((i - 32) % 8)));
  }
  return 0;
}
