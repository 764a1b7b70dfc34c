#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY: compiles the UNMODIFIED reference sources
# (/root/reference/proj/src/*.cpp, its CLI tools/relsim_main.cpp and its test
# suites tests/*.cpp) against the shims in oracle/ref_shim (eigen-lite,
# doctest-lite, CLI11-lite, a forward to the on-disk nlohmann json), plus the
# dump driver oracle/ref_driver.cpp.  Outputs only into oracle/_ref/ (git-ignored;
# travels to the GPU box with the snapshot).  Never reads or writes anything
# else under /root/reference.  usage: oracle/ref_build.sh [-j N]
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${RELSIM_REF:-/root/reference/proj}"
OUT="$HERE/_ref"
JOBS="${JOBS:-$(nproc)}"
if [ ! -d "$REF/src" ]; then
  echo "ref_build: $REF not present (the reference only exists in the build container)" >&2
  exit 0
fi
JSON_INC=""
for d in /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty \
         /usr/include /usr/local/include; do
  if [ -f "$d/nlohmann/json.hpp" ]; then JSON_INC="$d"; break; fi
done
if [ -z "$JSON_INC" ]; then echo "ref_build: nlohmann/json.hpp not found" >&2; exit 1; fi
mkdir -p "$OUT/obj"
CXX="${CXX:-g++}"
FLAGS=(-std=c++20 -O2 -fPIC -w -I"$HERE/ref_shim" -I"$JSON_INC" -I"$REF/include" -I"$REF/tests"
       -DRELSIM_SCENES_DIR="\"$REF/scenes\"" -pthread)
objs=()
pids=()
for f in "$REF"/src/*.cpp; do
  o="$OUT/obj/$(basename "${f%.cpp}").o"
  objs+=("$o")
  if [ ! -f "$o" ] || [ "$f" -nt "$o" ] || [ "$HERE/ref_shim/Eigen/Dense" -nt "$o" ]; then
    "$CXX" "${FLAGS[@]}" -c "$f" -o "$o" &
    pids+=($!)
    if [ "${#pids[@]}" -ge "$JOBS" ]; then wait "${pids[0]}"; pids=("${pids[@]:1}"); fi
  fi
done
for p in "${pids[@]}"; do wait "$p"; done
ar rcs "$OUT/librelsim.a" "${objs[@]}"
"$CXX" "${FLAGS[@]}" "$REF/tools/relsim_main.cpp" "$OUT/librelsim.a" -o "$OUT/relsim"
"$CXX" "${FLAGS[@]}" "$HERE/ref_driver.cpp" "$OUT/librelsim.a" -o "$OUT/ref_driver"
if [ "${1:-}" = "--tests" ]; then
  pids=()
  for t in "$REF"/tests/test_*.cpp; do
    "$CXX" "${FLAGS[@]}" "$t" "$OUT/librelsim.a" -o "$OUT/$(basename "${t%.cpp}")" &
    pids+=($!)
    if [ "${#pids[@]}" -ge "$JOBS" ]; then wait "${pids[0]}"; pids=("${pids[@]:1}"); fi
  done
  for p in "${pids[@]}"; do wait "$p"; done
fi
echo "ref_build: $OUT"
