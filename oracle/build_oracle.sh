#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY: builds the C restatement (oracle/oracle.c) as a float and a double
# library under oracle/_build/ (git-ignored). -ffp-contract=off keeps multiply and add separate,
# matching the reference's canonical (no -march) build.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
mkdir -p "$HERE/_build"
gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared "$HERE/oracle.c" -o "$HERE/_build/liboracle_f32.so" -lm
gcc -std=c11 -O2 -ffp-contract=off -fPIC -shared -DOR_S=double -DOR_F64 "$HERE/oracle.c" -o "$HERE/_build/liboracle_f64.so" -lm
echo "built $HERE/_build/liboracle_{f32,f64}.so"
