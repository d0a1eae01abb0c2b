#!/usr/bin/env bash
# Build libghostx variants with extra -D flags into build/variants/<tag>.so
#   build_variants.sh "tag1:-DFOO=1 -DBAR=2" "tag2:..."
set -e
cd "$(dirname "$0")/.."
mkdir -p build/variants
C=paper_2403_12179_b200/csrc
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
    -I include -I $C -cudart static $flags -o build/variants/$tag.so $C/*.cpp $C/*.cu &
done
wait
ls build/variants
