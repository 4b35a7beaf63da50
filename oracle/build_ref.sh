#!/usr/bin/env bash
# Compiles the reference wgtune library (the tuner side of the path: space,
# features, synthgen, simoracle, datastore, learn, tuner, bench) directly from
# its sources under /root/reference — no CMake, no copies into this repo —
# into oracle/_ref/ (git-ignored; travels to the GPU box as built files).
# Used only by tests/ as the parity checker for the host C++ tuner.
#
# Third-party: nlohmann/json (unpinned by the reference, vendor/ is absent;
# we use the 3.11.3 copy shipped in this image under cudnn_frontend).
# serve.cpp (TCP daemon, out of scope) is excluded.
set -euo pipefail
REF=/root/reference/proj
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
JSON_INC=/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty
CXX=${CXX:-g++}
[ -d "$REF/src" ] || { echo "reference sources not present; skipping"; exit 0; }
mkdir -p "$OUT/obj"
SRCS="space scenario features synthgen simoracle datastore learn tuner bench"
stamp="$OUT/libwgtune_ref.a"
need=0
for s in $SRCS; do
  [ "$stamp" -nt "$REF/src/$s.cpp" ] || need=1
done
[ -f "$stamp" ] || need=1
if [ "$need" = 1 ]; then
  for s in $SRCS; do
    $CXX -std=c++20 -O2 -fPIC -I"$REF/include" -I"$JSON_INC" -c "$REF/src/$s.cpp" -o "$OUT/obj/$s.o" &
  done
  wait
  rm -f "$stamp"
  ar rcs "$stamp" "$OUT"/obj/*.o
fi
echo "$OUT/libwgtune_ref.a"

# Tuner-side parity harness (tests/parity/tuner_parity.cpp): links the
# reference library and the framework's libwgtb side by side.
REPO="$(cd "$HERE/.." && pwd)"
LIBDIR="$REPO/paper_1511_02490_b200/lib"
HARNESS="$OUT/tuner_parity"
if [ -f "$LIBDIR/libwgtb.so" ] && { [ ! -f "$HARNESS" ] || [ "$REPO/tests/parity/tuner_parity.cpp" -nt "$HARNESS" ] || [ "$LIBDIR/libwgtb.so" -nt "$HARNESS" ] || [ "$stamp" -nt "$HARNESS" ]; }; then
  $CXX -std=c++20 -O2 -I"$REF/include" -I"$REPO/include" -I"$JSON_INC" -I/usr/local/cuda/include \
    "$REPO/tests/parity/tuner_parity.cpp" -o "$HARNESS" "$stamp" \
    -L"$LIBDIR" -lwgtb -lsk_stencil -L/usr/local/cuda/lib64 -lcudart -pthread \
    -Wl,-rpath,"$LIBDIR" -Wl,-rpath,/usr/local/cuda/lib64
fi
echo "$HARNESS"

# The reference-side B200 binding (integration/b200_backend.cpp, INTEGRATION.md
# §2) linked into the reference's own collect(): simoracle.cpp is compiled
# without inlining and its run / kernel_max_wgsize / is_refused are weakened,
# so the binding's strong definitions replace the simulator while collect()
# and scenario_context() remain the reference's code.
BIN2="$OUT/b200_collect"
if [ -f "$LIBDIR/libsk_stencil.so" ] && { [ ! -f "$BIN2" ] || [ "$REPO/integration/b200_backend.cpp" -nt "$BIN2" ] || [ "$REPO/tests/parity/b200_collect_main.cpp" -nt "$BIN2" ] || [ "$LIBDIR/libsk_stencil.so" -nt "$BIN2" ]; }; then
  $CXX -std=c++20 -O0 -fno-inline -fPIC -I"$REF/include" -I"$JSON_INC" -c "$REF/src/simoracle.cpp" -o "$OUT/obj_simoracle_weak.o"
  syms=$(nm "$OUT/obj_simoracle_weak.o" | awk '$2=="T"{print $3}' | grep -E '^_ZN6wgtune(3run|17kernel_max_wgsize|10is_refused)E')
  args=""; for s in $syms; do args="$args --weaken-symbol=$s"; done
  objcopy $args "$OUT/obj_simoracle_weak.o"
  others=""; for s in space scenario features synthgen datastore learn tuner bench; do others="$others $OUT/obj/$s.o"; done
  $CXX -std=c++20 -O2 -I"$REF/include" -I"$REPO/include" -I"$JSON_INC" -I/usr/local/cuda/include \
    "$REPO/tests/parity/b200_collect_main.cpp" "$REPO/integration/b200_backend.cpp" "$OUT/obj_simoracle_weak.o" $others \
    -o "$BIN2" -L"$LIBDIR" -lsk_stencil -L/usr/local/cuda/lib64 -lcudart -pthread \
    -Wl,-rpath,"$LIBDIR" -Wl,-rpath,/usr/local/cuda/lib64
fi
echo "$BIN2"

# The reference's evaluate() on B200 sweep files (tests/parity/ref_evaluate.cpp).
BIN3="$OUT/ref_evaluate"
if [ ! -f "$BIN3" ] || [ "$REPO/tests/parity/ref_evaluate.cpp" -nt "$BIN3" ] || [ "$stamp" -nt "$BIN3" ]; then
  $CXX -std=c++20 -O2 -I"$REF/include" -I"$JSON_INC" "$REPO/tests/parity/ref_evaluate.cpp" -o "$BIN3" "$stamp" -pthread
fi
echo "$BIN3"
