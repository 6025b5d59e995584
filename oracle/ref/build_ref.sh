#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY.  Compiles the reference's own integer/bitstream
# translation units verbatim from /root/reference/proj/src (read-only; nothing
# is copied into the repo) into oracle/_ref/libtucomp_ref.so, with the
# reference's Release flags (-O3, no -march; the AVX2 TU gets -mavx2 -mfma,
# which its _mm256_fmadd_pd calls need).  Eigen is replaced by a forward-
# declaration stub (those TUs only name the Matrix<T> alias), tensor.cpp's
# Eigen-free helpers by tensor_min.cpp.  The FP half (sthosvd, factor_codec,
# pipeline) needs real Eigen and is NOT built; the oracle restates it.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${TUCOMP_REFERENCE:-/root/reference/proj}"
OUT="$HERE/../_ref"
if [ ! -d "$REF/src" ]; then
  echo "reference sources not present at $REF; skipping _ref build" >&2
  exit 0
fi
mkdir -p "$OUT/obj"
CXX="${CXX:-g++}"
FLAGS="-std=c++20 -O3 -DNDEBUG -fPIC -fopenmp -I$REF/include -I$HERE/eigen_stub -I$HERE"
for f in core_codec entropy error_model vectorize container kernels; do
  $CXX $FLAGS -c "$REF/src/$f.cpp" -o "$OUT/obj/$f.o"
done
$CXX $FLAGS -mavx2 -mfma -c "$REF/src/kernels_avx2.cpp" -o "$OUT/obj/kernels_avx2.o"
$CXX $FLAGS -c "$HERE/tensor_min.cpp" -o "$OUT/obj/tensor_min.o"
$CXX $FLAGS -c "$HERE/ref_shim.cpp" -o "$OUT/obj/ref_shim.o"
$CXX -shared -o "$OUT/libtucomp_ref.so" "$OUT"/obj/*.o -L/usr/lib/gcc/x86_64-linux-gnu/13 -lgomp
echo "built $OUT/libtucomp_ref.so"
