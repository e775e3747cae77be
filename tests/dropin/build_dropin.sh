#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Builds tests/dropin/_build/dropin_main: the reference's callers (extracted from
# /root/reference at build time by extract.py, never committed) compiled unchanged against
# include/mggcn/rowgcn.hpp and linked with libmggcn.so. Exit 3 when the reference is absent (GPU box):
# the prebuilt binary travels with the snapshot like the other in-tree build outputs.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
ROOT="$(cd "$HERE/../.." && pwd)"
JSON_DIR="${MGGCN_NLOHMANN_DIR:-/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann}"
python "$HERE/extract.py" "${MGGCN_REFERENCE:-/root/reference}" || exit $?
LIB="$ROOT/paper_2110_08688_b200"
g++ -std=gnu++20 -O2 -Wall -Wno-unused-function -I "$ROOT/include" -I "$JSON_DIR" -I "$HERE" \
    "$HERE/dropin_main.cpp" -L "$LIB" -lmggcn -Wl,-rpath,'$ORIGIN/../../../paper_2110_08688_b200' \
    -o "$HERE/_build/dropin_main.tmp"
mv "$HERE/_build/dropin_main.tmp" "$HERE/_build/dropin_main"
echo "built $HERE/_build/dropin_main"
