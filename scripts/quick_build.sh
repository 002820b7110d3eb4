#!/bin/bash
# Incremental parallel build of libcuhallar.so (the build() recipe), plus ptxas
# register/stack stats of both persistent kernels.
cd "$(dirname "$0")/.."
python -c "import __graft_entry__ as g; g.build()" 2>&1 | grep -E "error|warning" | head -30
for o in paper_2505_13719_b200/build/*.cu.o; do
  cuobjdump -res-usage "$o" 2>/dev/null | grep -A1 -E "hallar_kernel|hallar_parity_kernel" | grep -E "REG|Function" | head -4
done
