#!/bin/bash
# Compile libcuhallar.so with the build() flags (+ ptxas stats) and install it in-tree.
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false \
  -Xcompiler -fPIC,-ffp-contract=off,-O3 -shared paper_2505_13719_b200/csrc/capi.cu \
  paper_2505_13719_b200/csrc/host_instances.cpp -o /tmp/quick.so -Xptxas -v 2>&1 \
  | grep -E "error|warning|_ZN6hallar13hallar_kernel" -A3 | head -30
[ -f /tmp/quick.so ] && cp /tmp/quick.so paper_2505_13719_b200/libcuhallar.so && rm /tmp/quick.so && \
  python -c "import __graft_entry__ as g; open(g.STAMP, 'w').write(g._digest())" && echo installed
