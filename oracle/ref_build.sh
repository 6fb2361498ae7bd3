#!/usr/bin/env bash
# Probe whether the reference's hot-path sources can be compiled directly
# with g++ (no cmake). They cannot in this image: every header includes
# <Eigen/Dense> (proj/CMakeLists.txt:13-18) and Eigen3 is absent, as are the
# vendored doctest/json/CLI11 headers (proj/.gitignore:2). The probe writes
# its verdict to oracle/_ref/STATUS; nothing else is produced.
set -u
HERE="$(cd "$(dirname "$0")" && pwd)"
OUT="$HERE/_ref"
mkdir -p "$OUT"
REF=/root/reference/proj
if [ ! -d "$REF" ]; then
  echo "reference not present" > "$OUT/STATUS"; exit 0
fi
for inc in /usr/include/eigen3 /usr/local/include/eigen3 /usr/include/Eigen; do
  if [ -e "$inc" ]; then
    if g++ -O3 -std=c++20 -fPIC -shared -I"$REF/include" -I"$inc" -I"$REF/src" \
        "$REF"/src/{common,kernels,geometry,chebyshev,tt,farfield,nearfield,phmatrix}.cpp \
        -o "$OUT/libphmat_ref.so" 2> "$OUT/build.log"; then
      echo "built with $inc" > "$OUT/STATUS"; exit 0
    fi
  fi
done
echo "unbuildable: Eigen3 headers not found (reference hard dependency)" > "$OUT/STATUS"
exit 0
