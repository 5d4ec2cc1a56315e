#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Builds the two oracle libraries into oracle/_ref/:
#   libgeoheat_port.so  the C restatement (oracle/geoheat_oracle.c); always built.
#   libgh_meshgen.so    the seeded BASELINE workload generators (workloads/meshgen.c),
#                       so bench.py's CPU reference arm maps no product library.
#   libgeoheat_ref.so   the unmodified reference headers compiled in place from
#                       /root/reference/proj/{include,tests} with the Eigen shim;
#                       built only when /root/reference exists (this container).
# Flags follow the reference build (proj/CMakeLists.txt: C++20, -O2, OpenMP) and
# pin FMA off so the bits match SURVEY.md §8(c): no -march, -ffp-contract=off.
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
out="$here/_ref"
mkdir -p "$out"
REF="${GEOHEAT_REFERENCE:-/root/reference/proj}"

gcc -std=gnu11 -O2 -DNDEBUG -fopenmp -ffp-contract=off -fPIC -shared \
    -o "$out/libgeoheat_port.so.tmp" "$here/geoheat_oracle.c" -lm
mv "$out/libgeoheat_port.so.tmp" "$out/libgeoheat_port.so"

gcc -std=gnu11 -O2 -fPIC -shared -ffp-contract=off \
    -o "$out/libgh_meshgen.so.tmp" "$here/../workloads/meshgen.c" -lm
mv "$out/libgh_meshgen.so.tmp" "$out/libgh_meshgen.so"

if [ -d "$REF/include/geoheat" ]; then
  g++ -std=gnu++20 -O2 -DNDEBUG -fopenmp -ffp-contract=off -fPIC -shared \
      -I"$here/eigen_shim" -I"$REF/include" -I"$REF/tests" -I"$here" \
      -o "$out/libgeoheat_ref.so.tmp" "$here/ref_driver.cpp"
  mv "$out/libgeoheat_ref.so.tmp" "$out/libgeoheat_ref.so"
else
  echo "build_ref.sh: $REF absent; keeping any prebuilt libgeoheat_ref.so" >&2
fi
