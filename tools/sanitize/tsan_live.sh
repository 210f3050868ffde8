#!/bin/bash
# TSan build of the live-mode host runtime (timed backend) + the pure-C++
# pieces it uses; the CUDA-side symbols resolve to libdualpath.so (never
# called on the timed backend).  Usage: bash tools/sanitize/tsan_live.sh [out.log]
set -e
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
OUT=${1:-/tmp/tsan_live.log}
SRC=$ROOT/paper_2602_21548_b200/csrc
g++ -std=c++20 -O1 -g -fsanitize=thread -ffp-contract=off -I$ROOT/include -I/usr/local/cuda/include \
  $ROOT/tools/sanitize/tsan_live.cpp $SRC/live.cpp $SRC/nic.cpp $SRC/scheduler.cpp $SRC/types.cpp \
  $SRC/workload.cpp -L$ROOT/paper_2602_21548_b200 -ldualpath -Wl,-rpath,$ROOT/paper_2602_21548_b200 \
  -L/usr/local/cuda/lib64 -lcudart -lpthread -o /tmp/tsan_live
TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1" /tmp/tsan_live > "$OUT" 2>&1
rc=$?
grep -c "WARNING: ThreadSanitizer" "$OUT" || true
exit $rc
