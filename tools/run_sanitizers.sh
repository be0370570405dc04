#!/usr/bin/env bash
# compute-sanitizer over every libffx kernel (tools/sanitize_paths.c) on a
# small ragged payload.  Logs: ${OUT:-gpurun_out/r2}/sanitizer_<tool>.log
set -u
cd "$(dirname "$0")/.."
OUT=${OUT:-gpurun_out/r2}
mkdir -p "$OUT"
gcc -std=c99 -O2 -Iinclude tools/sanitize_paths.c -Lpaper_2512_03644_b200 -lffx \
    -Wl,-rpath,"$PWD/paper_2512_03644_b200" -o tools/sanitize_paths || exit 1
./tools/sanitize_paths > "$OUT/sanitizer_plain.log" 2>&1; echo "plain rc=$?" >> "$OUT/sanitizer_plain.log"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check full"
  timeout 900 compute-sanitizer --tool "$tool" $extra --print-limit 50 ./tools/sanitize_paths \
      > "$OUT/sanitizer_$tool.log" 2>&1
  echo "rc=$?" >> "$OUT/sanitizer_$tool.log"
done
