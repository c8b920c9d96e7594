#!/usr/bin/env bash
# Builds tests/cpp/build/facade_test against the reference headers + TUs (oracle/_ref)
# and libsfctr_b200.so. Needs /root/reference (build container only); the binary then
# travels to the GPU box with the snapshot.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
REF="${SFCTR_REFERENCE:-/root/reference}/proj/core/include"
[ -d "$REF" ] && [ -f "$ROOT/oracle/_ref/libsfctr_ref.so" ] || { echo "reference absent; skip"; exit 0; }
mkdir -p "$HERE/build"
g++ -std=c++20 -O1 -Wall -I"$ROOT/include" -I"$REF" "$HERE/facade_test.cpp" \
    -L"$ROOT/oracle/_ref" -lsfctr_ref -L"$ROOT/paper_2104_08542_b200" -l:libsfctr_b200.so \
    -Wl,-rpath,'$ORIGIN/../../../oracle/_ref' -Wl,-rpath,'$ORIGIN/../../../paper_2104_08542_b200' \
    -o "$HERE/build/facade_test"
echo "built $HERE/build/facade_test"
