#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Compiles the unmodified reference (rowgcn) headers in place from
# /root/reference/proj into oracle/_ref/librowgcn_ref.so through oracle/ref_shim.cpp, using the
# reference's own Release flags (proj/CMakeLists.txt: C++20, -O3 -DNDEBUG, no -march => no FMA
# contraction). The reference's CMake build system is NOT run; its single non-template
# source (proj/src/collectives.cpp) is compiled directly where it lies. Output goes only to
# oracle/_ref/ (git-ignored, travels to the GPU box with the snapshot).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${MGGCN_REFERENCE:-/root/reference}"
JSON_DIR="${MGGCN_NLOHMANN_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
if [ ! -d "$REF/proj/include/rowgcn" ]; then
  echo "build_ref.sh: reference not present at $REF (expected on the build container only)" >&2
  exit 3
fi
mkdir -p "$HERE/_ref"
OUT="$HERE/_ref/librowgcn_ref.so"
g++ -std=gnu++20 -O3 -DNDEBUG -fPIC -shared -pthread \
    -I "$REF/proj/include" -I "$JSON_DIR" \
    "$HERE/ref_shim.cpp" "$REF/proj/src/collectives.cpp" \
    -o "$OUT.tmp"
mv "$OUT.tmp" "$OUT"
echo "built $OUT"
