# usage: bash scripts/ncu_pass.sh <tag> <instance> <kind> <s>   (one kernel: a bench_pass launch)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
cat > /tmp/ncu_one.py <<PY
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2505_13719_b200 as H
name, kind, s = sys.argv[1], sys.argv[2], int(sys.argv[3])
inst = (H.gen_matrix_completion(H.McSpec(400000, 600000, 3, seed=0)) if name == "C4"
        else H.build_theta_instance(H.make_hypercube(int(name[1:]))))
rng = np.random.default_rng(0)
U = rng.standard_normal((inst.n, s)); U /= np.linalg.norm(U)
p = rng.standard_normal(inst.m)
inst.bench_pass(kind, U, p, beta=10.0, iters=2)
print(inst.bench_pass(kind, U, p, beta=10.0, iters=20))
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hallar_kernel -s 1 -c 1 \
  -o /tmp/ncu_$1 python /tmp/ncu_one.py $2 $3 $4 > gpurun_out/ncu_$1.log 2>&1
# keep gpurun_out small (<= 64 MiB comes back): raw metrics + details as CSV, source hot spots
ncu -i /tmp/ncu_$1.ncu-rep --page raw --csv > gpurun_out/ncu_$1_raw.csv 2>/dev/null
ncu -i /tmp/ncu_$1.ncu-rep --page details --csv > gpurun_out/ncu_$1_details.csv 2>/dev/null
