"""DRAM-throughput timeline of one kernel from an ncu report's PM sampling
(`ncu --set full` captures it): steady-state level and the start / tail
deficits in microseconds of steady-state time.

    python tools/pm_timeline.py snap.ncu-rep
"""
import glob
import sys

sys.path.insert(0, (glob.glob("/opt/nvidia/nsight-compute/*/extras/python") or ["."])[0])
import ncu_report  # noqa: E402

M = "FBSP.TriageCompute.dram__throughput.avg.pct_of_peak_sustained_elapsed"


def main(path):
    a = ncu_report.load_report(path).range_by_idx(0).action_by_idx(0)
    m = a.metric_by_name(M)
    vals = [m.as_double(i) for i in range(m.num_instances())]
    corr = a.metric_by_name(M).correlation_ids()
    ts = [corr.as_uint64(i) for i in range(corr.num_instances())] if corr is not None else list(range(len(vals)))
    dur_us = a.metric_by_name("gpu__time_duration.sum").as_double() / 1e3
    # keep the samples inside the kernel (non-zero span)
    on = [i for i, v in enumerate(vals) if v > 1.0]
    lo, hi = on[0], on[-1]
    span = ts[hi] - ts[lo]
    per = (span / (hi - lo)) if hi > lo else 1
    body = sorted(vals[lo:hi + 1])
    steady = body[len(body) // 2]
    us = lambda n: n * per / 1e3 if per > 10 else n * dur_us / len(vals)
    n = hi - lo + 1
    q = max(1, n // 10)
    start = sum(max(0.0, steady - v) for v in vals[lo:lo + q]) / steady
    tail = sum(max(0.0, steady - v) for v in vals[hi - q + 1:hi + 1]) / steady
    print(f"samples {len(vals)} in-kernel {n}, sample period {us(1):.3f} us, kernel {dur_us:.1f} us")
    print(f"steady (median) {steady:.1f}% of DRAM peak")
    print(f"start deficit (first 10%) {us(start):.1f} us, tail deficit (last 10%) {us(tail):.1f} us")
    w = max(1, n // 40)
    for i in range(lo, hi + 1, w):
        seg = vals[i:i + w]
        print(f"{us(i - lo):8.1f} us  {sum(seg) / len(seg):6.1f}")


if __name__ == "__main__":
    main(sys.argv[1])
