// ffx_standby.cpp -- the replacement process of a failed rank, and the two
// processes around it, over libffx's C ABI only (no Python, no torch).
//
// Reference flow being timed: Controller::orchestrate_recovery
// (controller.cpp:307-322) -> plan_recovery (:144-209) -> the holder's
// NeighborBuffer::framed_at (ckpt.cpp:95-100) -> StateForward to the
// substitute -> assemble_restore (ckpt.cpp:140-167).  On a B200 node the
// substitute is a fresh process (or a pre-started warm spare) that maps the
// holder's replica over CUDA IPC and pulls + verifies the state itself.
//
//   ffx_standby holder  --device D --d N --phi P --origin DP --capacity B --versions V --store DIR
//       creates the replica it holds for ring predecessor DP, publishes its
//       handle in DIR (write + rename), prints "READY", waits for EOF on stdin.
//   ffx_standby origin  --device D --d N --phi P --role DP --store DIR --holder H
//                       --regions SPEC [--regions2 SPEC]
//       allocates + materializes its state registry on the device, snapshots
//       iteration 1 (and 2 from --regions2) into holder H's replica, prints
//       "SNAPSHOTTED <it>", waits (the harness SIGKILLs it).
//   ffx_standby standby --device D --d N --phi P --role DP --store DIR
//                       (--warm [--prealloc B] | --t0 NS) [--target IT] [--samples FILE] [--check]
//       --warm: a provisioned spare -- CUDA context + ffx ctx, peer access to
//       every NVLink peer, and (--prealloc) the job's state arena allocated
//       before the failure; prints "ARMED", then reads "FAIL <t0 ns>" on
//       stdin.  --t0: a cold start after the failure.
//       Then: plan_recovery -> open the planned holder's replica handle ->
//       allocate + register the regions the committed slot records ->
//       ffx_recover (gather + per-slice FNV verify) -> one JSON line with the
//       time from the failure notice (CLOCK_MONOTONIC t0) to verified state
//       and its breakdown.  --check (untimed): blob_is_sound per region on the
//       device; --samples: head / tail of every region to FILE for the oracle.
//
// SPEC = comma-separated kind:bytes:HEX64 (materialize(digest, bytes)) or
// kind:bytes:=HEX (literal bytes, for the cursor / RNG words).
#include <fcntl.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <cerrno>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>
#include <vector>

#include "ffx.h"

namespace {

uint64_t now_ns() {
  timespec ts{};
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return static_cast<uint64_t>(ts.tv_sec) * 1000000000ull + static_cast<uint64_t>(ts.tv_nsec);
}

[[noreturn]] void die(const char* what, int st) {
  std::fprintf(stderr, "ffx_standby: %s failed (%d): %s\n", what, st, ffx_last_error());
  std::exit(3);
}
void ck(int st, const char* what) {
  if (st != FFX_OK) die(what, st);
}

struct Args {
  std::string mode, store, regions, regions2, samples;
  int device = 0, origin = -1, role = -1, holder = -1;
  uint32_t d = 2, versions = 2;
  uint64_t phi = 0, capacity = 0, t0 = 0, slice = 4096, target = 0, prealloc = 0;
  bool warm = false, check = false, shared = false, touch = false;
  int repeat = 0;
};

Args parse(int argc, char** argv) {
  Args a;
  if (argc < 2) {
    std::fprintf(stderr, "usage: ffx_standby holder|origin|standby [options]\n");
    std::exit(2);
  }
  a.mode = argv[1];
  for (int i = 2; i < argc; ++i) {
    const std::string k = argv[i];
    auto val = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "ffx_standby: %s needs a value\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--device") a.device = std::atoi(val().c_str());
    else if (k == "--d") a.d = static_cast<uint32_t>(std::strtoul(val().c_str(), nullptr, 10));
    else if (k == "--phi") a.phi = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--origin") a.origin = std::atoi(val().c_str());
    else if (k == "--role") a.role = std::atoi(val().c_str());
    else if (k == "--holder") a.holder = std::atoi(val().c_str());
    else if (k == "--capacity") a.capacity = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--versions") a.versions = static_cast<uint32_t>(std::strtoul(val().c_str(), nullptr, 10));
    else if (k == "--slice") a.slice = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--store") a.store = val();
    else if (k == "--regions") a.regions = val();
    else if (k == "--regions2") a.regions2 = val();
    else if (k == "--samples") a.samples = val();
    else if (k == "--prealloc") a.prealloc = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--target") a.target = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--t0") a.t0 = std::strtoull(val().c_str(), nullptr, 10);
    else if (k == "--warm") a.warm = true;
    else if (k == "--check") a.check = true;
    else if (k == "--shared") a.shared = true;
    else if (k == "--touch") a.touch = true;
    else if (k == "--repeat") a.repeat = std::atoi(val().c_str());
    else {
      std::fprintf(stderr, "ffx_standby: unknown option %s\n", k.c_str());
      std::exit(2);
    }
  }
  return a;
}

ffx_cluster_spec spec_of(const Args& a) {
  ffx_cluster_spec s{};
  s.num_nodes = 1;
  s.gpus_per_node = a.d;
  s.data_parallel = a.d;
  s.pipeline_parallel = 1;
  s.tensor_parallel = 1;
  s.distributed_optimizer = 1;
  s.params_per_device = a.phi;
  return s;
}

ffx_role dp_role(int dp) { return ffx_role{static_cast<uint16_t>(dp), 0, 0}; }

// The handle store: one file per (origin, holder) pair, published atomically.
std::string handle_path(const std::string& dir, int origin, int holder) {
  return dir + "/replica_o" + std::to_string(origin) + "_h" + std::to_string(holder) + ".ffxh";
}

void publish(const std::string& path, const uint8_t* data, size_t n) {
  const std::string tmp = path + ".tmp";
  const int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC | O_CLOEXEC, 0600);
  if (fd < 0 || ::write(fd, data, n) != static_cast<ssize_t>(n) || ::fsync(fd) != 0) {
    std::fprintf(stderr, "ffx_standby: cannot write %s: %s\n", tmp.c_str(), std::strerror(errno));
    std::exit(3);
  }
  ::close(fd);
  if (::rename(tmp.c_str(), path.c_str()) != 0) {
    std::fprintf(stderr, "ffx_standby: rename %s: %s\n", path.c_str(), std::strerror(errno));
    std::exit(3);
  }
}

bool fetch(const std::string& path, uint8_t* data, size_t n) {
  const int fd = ::open(path.c_str(), O_RDONLY | O_CLOEXEC);
  if (fd < 0) return false;
  const bool ok = ::read(fd, data, n) == static_cast<ssize_t>(n);
  ::close(fd);
  return ok;
}

int hexval(char c) {
  if (c >= '0' && c <= '9') return c - '0';
  if (c >= 'a' && c <= 'f') return c - 'a' + 10;
  if (c >= 'A' && c <= 'F') return c - 'A' + 10;
  return -1;
}

std::vector<uint8_t> unhex(const std::string& h) {
  std::vector<uint8_t> out;
  if (h.size() % 2) return out;
  for (size_t i = 0; i < h.size(); i += 2) {
    const int a = hexval(h[i]), b = hexval(h[i + 1]);
    if (a < 0 || b < 0) return {};
    out.push_back(static_cast<uint8_t>(a * 16 + b));
  }
  return out;
}

struct RegionSpec {
  int kind;
  uint64_t bytes;
  std::vector<uint8_t> digest;   // materialize(digest, bytes), or
  std::vector<uint8_t> literal;  // exactly these bytes
};

std::vector<RegionSpec> parse_regions(const std::string& s) {
  std::vector<RegionSpec> out;
  size_t pos = 0;
  while (pos < s.size()) {
    size_t end = s.find(',', pos);
    if (end == std::string::npos) end = s.size();
    const std::string item = s.substr(pos, end - pos);
    pos = end + 1;
    const size_t c1 = item.find(':'), c2 = item.find(':', c1 + 1);
    if (c1 == std::string::npos || c2 == std::string::npos) {
      std::fprintf(stderr, "ffx_standby: bad region spec '%s'\n", item.c_str());
      std::exit(2);
    }
    RegionSpec r;
    r.kind = std::atoi(item.substr(0, c1).c_str());
    r.bytes = std::strtoull(item.substr(c1 + 1, c2 - c1 - 1).c_str(), nullptr, 10);
    const std::string v = item.substr(c2 + 1);
    if (!v.empty() && v[0] == '=') {
      r.literal = unhex(v.substr(1));
      if (r.literal.size() != r.bytes) {
        std::fprintf(stderr, "ffx_standby: literal region of %zu bytes, declared %llu\n", r.literal.size(),
                     (unsigned long long)r.bytes);
        std::exit(2);
      }
    } else {
      r.digest = unhex(v);
      if (r.digest.size() != 32 || r.bytes < 32) {
        std::fprintf(stderr, "ffx_standby: region needs a 32-byte digest and >= 32 bytes\n");
        std::exit(2);
      }
    }
    out.push_back(std::move(r));
  }
  return out;
}

void fill(void* dev, const RegionSpec& r) {
  if (!r.literal.empty()) ck(ffx_memcpy(dev, r.literal.data(), r.bytes, nullptr, 1), "literal region H2D");
  else ck(ffx_materialize(dev, r.digest.data(), r.bytes, nullptr), "materialize");
}

void wait_stdin_eof() {
  std::string line;
  while (std::getline(std::cin, line))
    if (line == "QUIT") break;
}

// ---- holder -----------------------------------------------------------------

int run_holder(const Args& a) {
  const ffx_cluster_spec spec = spec_of(a);
  ffx_ctx* ctx = nullptr;
  ffx_role self{};
  ck(ffx_dp_neighbor(&spec, dp_role(a.origin), &self), "dp_neighbor");
  ck(ffx_open(a.device, &spec, self, a.slice, &ctx), "open");
  ffx_replica* rep = nullptr;
  // --shared: a VMM (cuMemCreate) allocation exported by fd, mapped with 2 MiB
  // pages in the importer; default: cudaMalloc + CUDA IPC
  if (a.shared) ck(ffx_replica_create_shared(ctx, dp_role(a.origin), a.capacity, a.versions, &rep), "create_shared");
  else ck(ffx_replica_create(ctx, dp_role(a.origin), a.capacity, a.versions, &rep), "replica_create");
  uint8_t h[FFX_HANDLE_BYTES];
  ck(ffx_replica_export(rep, h), "replica_export");
  publish(handle_path(a.store, a.origin, self.dp), h, sizeof h);
  std::printf("READY %d\n", self.dp);
  std::fflush(stdout);
  wait_stdin_eof();
  ffx_replica_destroy(rep);
  ffx_close(ctx);
  return 0;
}

// ---- origin -----------------------------------------------------------------

int run_origin(const Args& a) {
  const ffx_cluster_spec spec = spec_of(a);
  ffx_ctx* ctx = nullptr;
  ck(ffx_open(a.device, &spec, dp_role(a.role), a.slice, &ctx), "open");
  const std::vector<RegionSpec> regs = parse_regions(a.regions);
  const std::vector<RegionSpec> regs2 = a.regions2.empty() ? std::vector<RegionSpec>{} : parse_regions(a.regions2);
  std::vector<void*> dev(regs.size(), nullptr);
  for (size_t i = 0; i < regs.size(); ++i) {
    ck(ffx_device_alloc(a.device, regs[i].bytes, &dev[i]), "device_alloc");
    fill(dev[i], regs[i]);
    ck(ffx_register_region(ctx, regs[i].kind, dev[i], regs[i].bytes, 1), "register_region");
  }
  uint8_t h[FFX_HANDLE_BYTES];
  if (!fetch(handle_path(a.store, a.role, a.holder), h, sizeof h)) {
    std::fprintf(stderr, "ffx_standby: no handle for holder %d\n", a.holder);
    return 3;
  }
  ffx_replica* view = nullptr;
  ck(ffx_replica_open(ctx, h, &view), "replica_open");
  ck(ffx_snapshot_target(ctx, view), "snapshot_target");
  ck(ffx_snapshot(ctx, 1, nullptr, nullptr), "snapshot 1");
  uint64_t last = 1;
  if (!regs2.empty()) {
    // the optimizer step of iteration 2 rewrites the state in place
    for (size_t i = 0; i < regs.size() && i < regs2.size(); ++i) fill(dev[i], regs2[i]);
    ck(ffx_snapshot(ctx, 2, nullptr, nullptr), "snapshot 2");
    last = 2;
  }
  ck(ffx_stream_sync(nullptr), "sync");
  std::printf("SNAPSHOTTED %llu\n", (unsigned long long)last);
  std::fflush(stdout);
  wait_stdin_eof();  // the harness kills this process here
  return 0;
}

// A spare loads the gather/verify kernel before any failure (the first launch
// in a process pays the module load): one tiny copy + verify.
void warm_kernels(int device) {
  const uint64_t n = 1 << 16, s = 4096;
  void *a = nullptr, *b = nullptr, *sums = nullptr, *res = nullptr;
  ck(ffx_device_alloc(device, n, &a), "warm alloc");
  ck(ffx_device_alloc(device, n, &b), "warm alloc");
  ck(ffx_device_alloc(device, n / s * 8, &sums), "warm alloc");
  ck(ffx_device_alloc(device, 16, &res), "warm alloc");
  ck(ffx_expand(a, std::vector<uint8_t>(32, 1).data(), n, nullptr), "warm expand");
  ck(ffx_slice_checksums(a, n, s, static_cast<uint64_t*>(sums), nullptr), "warm checksums");
  ck(ffx_copy_verify(b, a, n, s, static_cast<const uint64_t*>(sums), static_cast<uint64_t*>(res), nullptr),
     "warm copy_verify");
  ck(ffx_stream_sync(nullptr), "warm sync");
  for (void* p : {a, b, sums, res}) ffx_device_free(device, p);
}

// ---- standby (the replacement) ----------------------------------------------

int run_standby(const Args& a) {
  const uint64_t t_main = now_ns();
  const ffx_cluster_spec spec = spec_of(a);
  const ffx_role me = dp_role(a.role);
  ffx_ctx* ctx = nullptr;
  void* arena = nullptr;  // --prealloc: regions are carved from it
  uint64_t t0 = a.t0, t_ctx_start = 0, t_ctx = 0;
  if (a.warm) {
    // a spare that starts before the failure: CUDA context + ffx ctx ready
    t_ctx_start = now_ns();
    ck(ffx_open(a.device, &spec, me, a.slice, &ctx), "open");
    ck(ffx_prepare_peers(a.device, nullptr), "prepare_peers");
    warm_kernels(a.device);
    if (a.prealloc) {
      ck(ffx_device_alloc(a.device, a.prealloc, &arena), "prealloc");
      // --touch: write the arena once while arming, so the restore's stores
      // meet memory the GPU has already touched
      if (a.touch) ck(ffx_expand(arena, std::vector<uint8_t>(32, 0).data(), a.prealloc, nullptr), "touch");
      if (a.touch) ck(ffx_stream_sync(nullptr), "sync");
    }
    t_ctx = now_ns();
    std::printf("ARMED\n");
    std::fflush(stdout);
    std::string line;
    while (std::getline(std::cin, line)) {
      if (line.rfind("FAIL ", 0) == 0) {
        t0 = std::strtoull(line.c_str() + 5, nullptr, 10);
        break;
      }
    }
    if (!t0) return 4;
  }
  const uint64_t t_notice = now_ns();  // warm: the notice arrived; cold: main() ran
  if (!ctx) {
    t_ctx_start = now_ns();
    ck(ffx_open(a.device, &spec, me, a.slice, &ctx), "open");  // CUDA context creation happens here
    t_ctx = now_ns();
  }
  // 1. plan (controller.cpp:144-209): which holder serves this role
  std::vector<uint32_t> pods(a.d);
  std::vector<ffx_role> roles(a.d), lazy(a.d);
  std::vector<ffx_forward> fw(a.d);
  std::vector<ffx_redundant_source> red(a.d);
  ffx_recovery_plan plan{};
  plan.capacity = a.d;
  plan.failed_pods = pods.data();
  plan.failed_roles = roles.data();
  plan.lazy_backup_targets = lazy.data();
  plan.forwards = fw.data();
  plan.redundant_from = red.data();
  // --target: the ledger's global consistent iteration (controller.cpp:93-98);
  // without it the holder's newest committed slot is the resume point.  (A
  // zero global iteration plans no forwards -- nothing recorded yet,
  // controller.cpp:175-176 -- so plan with 1 to learn the holder.)
  ck(ffx_plan_recovery(&spec, nullptr, 0, &me, 1, a.target ? a.target : 1, 0, 1, &plan), "plan_recovery");
  if (plan.kind != FFX_PLAN_NEIGHBOR || plan.n_forwards != 1) {
    std::fprintf(stderr, "ffx_standby: plan is not a neighbour restore\n");
    return 3;
  }
  const int holder = static_cast<int>(plan.forwards[0].holder_dp);
  const uint64_t t_plan = now_ns();
  // 2. the holder's replica (handle store -> CUDA IPC mapping)
  uint8_t h[FFX_HANDLE_BYTES];
  if (!fetch(handle_path(a.store, a.role, holder), h, sizeof h)) {
    std::fprintf(stderr, "ffx_standby: no handle for holder %d\n", holder);
    return 3;
  }
  ffx_replica* src = nullptr;
  ck(ffx_replica_open(ctx, h, &src), "replica_open");
  const uint64_t t_open = now_ns();
  uint64_t target = a.target;
  if (!target) ck(ffx_replica_newest(src, &target), "replica_newest");
  uint32_t versions = 0, slot = 0;
  ck(ffx_replica_slots(src, &versions), "replica_slots");
  for (uint32_t v = 0; v < versions; ++v) {
    ffx_slot_info si{};
    ck(ffx_replica_slot_info(src, v, &si), "slot_info");
    if (si.state == 2 && si.iteration == target) slot = v + 1;
  }
  if (!slot) {
    std::fprintf(stderr, "ffx_standby: holder %d has no committed snapshot of iteration %llu\n", holder,
                 (unsigned long long)target);
    return 3;
  }
  --slot;
  const uint64_t t_map = now_ns();
  // 3. fresh allocations shaped like the committed state registry
  uint32_t n = 0;
  int32_t kinds[FFX_MAX_REGIONS];
  uint64_t sizes[FFX_MAX_REGIONS];
  ck(ffx_replica_slot_regions(src, slot, &n, kinds, sizes), "slot_regions");
  std::vector<void*> dev(n, nullptr);
  uint64_t total = 0, carved = 0;
  for (uint32_t i = 0; i < n; ++i) {
    const uint64_t need = (sizes[i] + 255) / 256 * 256;
    if (arena && carved + need <= a.prealloc) {
      dev[i] = static_cast<uint8_t*>(arena) + carved;
      carved += need;
    } else {
      ck(ffx_device_alloc(a.device, sizes[i], &dev[i]), "device_alloc");
    }
    ck(ffx_register_region(ctx, kinds[i], dev[i], sizes[i], 1), "register_region");
    total += sizes[i];
  }
  const uint64_t t_alloc = now_ns();
  // 4. gather + verify (assemble_restore): every slice re-hashed vs the table
  ffx_recover_report rpt{};
  const int rst = ffx_recover(ctx, src, target, nullptr, &rpt);
  const uint64_t t_done = now_ns();
  if (rst != FFX_OK) die("recover", rst);

  // ---- untimed: the same gather again (warm caches / touched destination) ----
  std::vector<double> again;
  for (int k = 0; k < a.repeat; ++k) {
    ffx_recover_report r2{};
    ck(ffx_recover(ctx, src, target, nullptr, &r2), "recover (repeat)");
    again.push_back(r2.seconds * 1e3);
  }

  // ---- untimed checks for the harness -----------------------------------
  int sound = -1;
  if (a.check) {
    sound = 1;
    for (uint32_t i = 0; i < n; ++i) {
      if (sizes[i] < 32 || kinds[i] == FFX_REGION_CURSOR || kinds[i] == FFX_REGION_RNG) continue;
      uint64_t bad = 0;
      ck(ffx_blob_check(dev[i], sizes[i], &bad, nullptr), "blob_check");
      if (bad != ~0ull) sound = 0;
    }
  }
  if (!a.samples.empty()) {
    FILE* f = std::fopen(a.samples.c_str(), "wb");
    if (!f) die("samples file", FFX_EINVAL);
    std::vector<uint8_t> buf;
    for (uint32_t i = 0; i < n; ++i) {
      const uint64_t k = sizes[i] < 8192 ? sizes[i] : 4096;  // head + tail (whole region if small)
      const uint64_t offs[2] = {0, sizes[i] - k};
      for (int j = 0; j < (sizes[i] < 8192 ? 1 : 2); ++j) {
        buf.resize(k);
        ck(ffx_memcpy(buf.data(), static_cast<uint8_t*>(dev[i]) + offs[j], k, nullptr, 1), "sample D2H");
        std::fwrite(buf.data(), 1, k, f);
      }
    }
    std::fclose(f);
  }
  auto ms = [](uint64_t a0, uint64_t a1) { return (a1 - a0) * 1e-6; };
  std::printf(
      "{\"mode\": \"%s\", \"target_iteration\": %llu, \"holder_dp\": %d, \"bytes\": %llu, \"regions\": %u, "
      "\"time_to_restore_s\": %.6f, \"breakdown_ms\": {\"notice_to_main\": %.3f, \"context\": %.3f, "
      "\"plan\": %.3f, \"ipc_map\": %.3f, \"ipc_open\": %.3f, \"alloc_register\": %.3f, \"gather_verify\": %.3f, "
      "\"gather_verify_kernel\": %.3f}, \"warm_context_ms\": %.3f, \"bad_slices\": %llu, \"verified\": %s, "
      "\"blob_is_sound\": %d, \"gbs_kernel\": %.1f, \"repeat_kernel_ms\": [%s]}\n",
      a.warm ? "warm" : "cold", (unsigned long long)target, holder, (unsigned long long)total, n,
      (t_done - t0) * 1e-9, a.warm ? ms(t0, t_notice) : ms(t0, t_main), a.warm ? 0.0 : ms(t_ctx_start, t_ctx),
      ms(a.warm ? t_notice : t_ctx, t_plan), ms(t_plan, t_map), ms(t_plan, t_open), ms(t_map, t_alloc),
      ms(t_alloc, t_done),
      rpt.seconds * 1e3, a.warm ? ms(t_ctx_start, t_ctx) : 0.0, (unsigned long long)rpt.bad_slices,
      rpt.bad_slices == 0 ? "true" : "false", sound, rpt.seconds > 0 ? total / rpt.seconds / 1e9 : 0.0,
      [&] {
        std::string j;
        for (double v : again) j += (j.empty() ? "" : ", ") + std::to_string(v);
        return j;
      }().c_str());
  std::fflush(stdout);
  for (void* p : dev)
    if (!arena || p < arena || p >= static_cast<uint8_t*>(arena) + a.prealloc) ffx_device_free(a.device, p);
  if (arena) ffx_device_free(a.device, arena);
  ffx_replica_destroy(src);
  ffx_close(ctx);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  if (a.store.empty()) {
    std::fprintf(stderr, "ffx_standby: --store DIR is required\n");
    return 2;
  }
  if (a.mode == "holder") return run_holder(a);
  if (a.mode == "origin") return run_origin(a);
  if (a.mode == "standby") return run_standby(a);
  std::fprintf(stderr, "ffx_standby: unknown mode %s\n", a.mode.c_str());
  return 2;
}
