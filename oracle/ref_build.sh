#!/usr/bin/env bash
# Compiles the reference itself into oracle/_ref/ (TEST INFRASTRUCTURE ONLY):
#   libphmat_ref.so  = the unmodified proj/src/*.cpp + oracle/ref_driver.cpp
#                      (a C driver over the reference's public API),
#   tests/test_*     = the reference's own doctest suites (proj/tests/*.cpp),
# against two committed shims that stand in for the reference's absent
# third-party headers: oracle/eigen_shim/Eigen/Dense (Eigen3 is a hard
# dependency, proj/CMakeLists.txt:13-18, and is not installed) and
# oracle/doctest_shim/doctest.h (vendor/ is git-ignored upstream,
# proj/.gitignore:2). harness.cpp's nlohmann json.hpp is the copy shipped in
# the image (cudnn_frontend's third-party tree). Nothing is copied out of
# /root/reference. On the GPU box (no /root/reference) the prebuilt files that
# travel with the snapshot are used and this script only reports.
set -u
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
mkdir -p "$OUT"
REF=/root/reference/proj
if [ ! -d "$REF" ]; then
  if [ -f "$OUT/libphmat_ref.so" ]; then echo "prebuilt (reference sources absent here)"; else
    echo "reference not present and no prebuilt library" > "$OUT/STATUS"; fi
  exit 0
fi
PURE="$(python -c 'import sysconfig; print(sysconfig.get_paths()["purelib"])' 2>/dev/null)"
JSON="$PURE/include/cudnn_frontend/thirdparty/nlohmann"
[ -f "$JSON/json.hpp" ] || JSON=""
if make -s -C "$HERE" -f ref.mk -j"$(nproc)" REF="$REF" OUT=_ref JSON="$JSON" > "$OUT/build.log" 2>&1; then
  echo "built: unmodified $REF/src/*.cpp + ref_driver.cpp against oracle/eigen_shim (g++ -O3 -DNDEBUG -std=c++20)" > "$OUT/STATUS"
else
  echo "build failed (see oracle/_ref/build.log)" > "$OUT/STATUS"
  cat "$OUT/build.log" >&2
  exit 1
fi
