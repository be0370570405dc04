// ref_bench.cpp -- the reference CPU path timed as a plain native process
// (TEST INFRASTRUCTURE: bench.py's cpu_baseline leg).  One std::thread per
// ring rank runs the reference's own HostSnapshots::take + NeighborBuffer::
// store (+ assemble_restore) on a bounded sample through ref_ring_* in
// libftsim_ref.so; prints one JSON object with the per-iteration medians.
// A separate executable (not a Python child) keeps the reference library
// out of every Python process of the measured GPU run.
//
//   ref_bench <threads> <bytes_per_thread> <iterations>
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

extern "C" {
void* ref_ring_setup(int threads, std::uint64_t bytes);
int ref_ring_run(void* h, std::uint64_t iteration, double* secs);
void ref_ring_free(void* h);
}

static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  const size_t n = v.size();
  return n % 2 ? v[n / 2] : 0.5 * (v[n / 2 - 1] + v[n / 2]);
}

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: ref_bench <threads> <bytes_per_thread> <iterations>\n");
    return 2;
  }
  const int threads = std::atoi(argv[1]);
  const std::uint64_t bytes = std::strtoull(argv[2], nullptr, 10);
  const int iters = std::atoi(argv[3]);
  void* h = ref_ring_setup(threads, bytes);
  std::vector<double> take, store, restore, snap;
  double secs[5];
  for (int i = 0; i < iters; ++i) {
    if (ref_ring_run(h, static_cast<std::uint64_t>(i + 1), secs) != 0) {
      std::fprintf(stderr, "reference ring iteration failed\n");
      return 3;
    }
    take.push_back(secs[0]);
    store.push_back(secs[1]);
    restore.push_back(secs[2]);
    snap.push_back(secs[4]);
  }
  ref_ring_free(h);
  std::printf("{\"threads\": %d, \"bytes_per_thread\": %llu, \"iterations\": %d, \"take_s\": %.6f, "
              "\"store_s\": %.6f, \"restore_s\": %.6f, \"snapshot_s\": %.6f}\n",
              threads, static_cast<unsigned long long>(bytes), iters, median(take), median(store),
              median(restore), median(snap));
  return 0;
}
