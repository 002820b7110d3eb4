#!/bin/bash
# Round 2 (session 4): GPU suite, e2e fetch path, CTA split-weight sweep, bench line.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu_c.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_c.log
timeout 300 python scripts/e2e_c4.py > gpurun_out/e2e_c4_c.log 2>&1
for w in 16 32 128; do
  CUHALLAR_SPLIT_W=$w timeout 300 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/prof_c4_w$w.jsonl 2>&1
done
timeout 900 python bench.py > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
exit 0
