#!/usr/bin/env bash
# TEST INFRASTRUCTURE: compiles the reference's present C++ translation units
# in place from /root/reference (read-only; nothing is copied into the repo)
# together with oracle/ref_shim.cpp into oracle/_ref/libsfctr_ref.so.
#
# The reference's own CMake build is not used: it requires Eigen3
# (proj/core/CMakeLists.txt:1) and lists five missing sources
# (manager/model/worker_ops/pipeline/report, core/CMakeLists.txt:10-14).
# The seven present TUs need neither, so they are compiled directly.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${SFCTR_REFERENCE:-/root/reference}/proj/core"
OUT="$HERE/_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not present at $REF; skipping oracle/_ref build" >&2
  exit 0
fi
mkdir -p "$OUT"
SRCS="config.cpp generator.cpp criteo.cpp vsi.cpp host_store.cpp cache_buffer.cpp log.cpp"
ARGS=()
for s in $SRCS; do ARGS+=("$REF/src/$s"); done
g++ -std=c++20 -O2 -fPIC -shared -Wall -Wextra -I"$REF/include" \
    "${ARGS[@]}" "$HERE/ref_shim.cpp" -o "$OUT/libsfctr_ref.so.tmp"
mv "$OUT/libsfctr_ref.so.tmp" "$OUT/libsfctr_ref.so"
echo "built $OUT/libsfctr_ref.so"
