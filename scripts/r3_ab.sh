#!/bin/bash
# Round 2 (session 4): A/B of the row-ordered SELL map and the cost-balanced CTA split.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_ab.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_ab.log
for tag in default even_tiles edge_map baseline; do
  case $tag in
    default) envs="" ;;
    even_tiles) envs="CUHALLAR_EVEN_TILES=1" ;;
    edge_map) envs="CUHALLAR_NO_SELL_MAP=1" ;;
    baseline) envs="CUHALLAR_EVEN_TILES=1 CUHALLAR_NO_SELL_MAP=1" ;;
  esac
  env $envs timeout 300 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/prof_c4_$tag.jsonl 2>&1
  env $envs timeout 300 python scripts/bench_passes.py mc400000_600000_3 --s 3 --kinds map_pass grad_pass lanczos_matvec > gpurun_out/passes_c4_$tag.jsonl 2>&1
done
timeout 300 python scripts/bench_passes.py H23 --s 2 --kinds map_pass grad_pass lanczos_matvec > gpurun_out/passes_h23.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_ab.json 2> gpurun_out/bench_ab.err
timeout 300 python scripts/e2e_c4.py > gpurun_out/e2e_c4.log 2>&1
bash scripts/ncu_pass.sh grad_c4_bal C4 grad_pass 3
# whole-solve source-level profile of the C4 solve (one launch; stall samples per source line)
cat > /tmp/solve_once.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2505_13719_b200 as H
inst = H.gen_matrix_completion(H.McSpec(400000, 600000, 3, seed=0))
cfg = H.SolverConfig(eps=1e-5)
H.solve(inst, cfg, fetch=False)
r = H.solve(inst, cfg, fetch=False)
print(r.status, r.device_seconds, r.fista_iters)
PY
timeout 1200 ncu --section SourceCounters --section WarpStateStats --section MemoryWorkloadAnalysis --section SpeedOfLight \
  --import-source on --clock-control none -k regex:hallar_kernel -s 1 -c 1 -o /tmp/ncu_solve python /tmp/solve_once.py > gpurun_out/ncu_solve.log 2>&1
ncu -i /tmp/ncu_solve.ncu-rep --page source --csv --print-source cuda 2>/dev/null | gzip > gpurun_out/ncu_solve_source.csv.gz
ncu -i /tmp/ncu_solve.ncu-rep --page raw --csv > gpurun_out/ncu_solve_raw.csv 2>/dev/null
exit 0
