#!/usr/bin/env bash
# Builds the UNMODIFIED reference library (C++20, CPU-only) from its sources
# where they lie under /root/reference/proj, plus our extern "C" marshalling
# layer (oracle/ref/ref_capi.cpp) and an Eigen-subset shim (Eigen 3 is absent
# from this image).  Output: oracle/_ref/libmilo_ref.so.
# Test infrastructure only (oracle/README in oracle/milo_oracle.h).  The .so is
# git-ignored but travels to the GPU box with the gpurun snapshot; the GPU box
# has no /root/reference, so this script is a no-op there if the .so exists.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${MILO_REFERENCE:-/root/reference/proj}"
OUT="$HERE/_ref"
mkdir -p "$OUT"
if [ ! -d "$REF/src" ]; then
  if [ -f "$OUT/libmilo_ref.so" ]; then exit 0; fi
  echo "reference sources not found at $REF; oracle/_ref not built" >&2
  exit 1
fi
JSON_DIR="$(python3 -c 'import os,site;import glob;c=[p for s in site.getsitepackages() for p in glob.glob(os.path.join(s,"include/cudnn_frontend/thirdparty/nlohmann"))];print(c[0] if c else "")')"
CXXFLAGS="-std=c++20 -O3 -fPIC -I$REF/include -I$HERE/ref/eigen_shim -I$JSON_DIR"
OBJ="$OUT/obj"
mkdir -p "$OBJ"
for f in "$REF"/src/*.cpp; do
  g++ $CXXFLAGS -c "$f" -o "$OBJ/$(basename "$f" .cpp).o" &
done
g++ $CXXFLAGS -c "$HERE/ref/ref_capi.cpp" -o "$OBJ/ref_capi.o" &
wait
g++ -shared -o "$OUT/libmilo_ref.so" "$OBJ"/*.o -lpthread
rm -rf "$OBJ"
echo "built $OUT/libmilo_ref.so"
# INTEGRATION.md section 2 compiled: the reference's types / gemm_w3a16 beside the B200
# library through include/milo_b200.hpp (needs the B200 library built first)
B200="$HERE/../paper_2504_02658_b200/lib/libmilo_b200.so"
if [ -f "$B200" ]; then
  g++ $CXXFLAGS -I"$HERE/../include" "$HERE/ref/b200_binding_check.cpp" "$OUT/libmilo_ref.so" "$B200" \
    -Wl,-rpath,'$ORIGIN' -Wl,-rpath,'$ORIGIN/../../paper_2504_02658_b200/lib' -o "$OUT/b200_binding_check"
  echo "built $OUT/b200_binding_check"
fi
