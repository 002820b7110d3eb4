#!/bin/bash
# Round 2 (session 4) final pass: GPU suite, bench line + reference arm, launch list,
# pass timings at C4 / H(23,2), ncu of the theta map.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_final.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_final.log
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref_final.json 2>> gpurun_out/bench_final.err
timeout 300 python scripts/bench_passes.py H23 --s 2 --kinds map_pass grad_pass lanczos_matvec > gpurun_out/passes_h23_final.jsonl 2>&1
CUHALLAR_NO_SELL_MAP=1 timeout 300 python scripts/bench_passes.py H23 --s 2 --kinds map_pass > gpurun_out/passes_h23_edgemap.jsonl 2>&1
timeout 300 python scripts/bench_passes.py mc400000_600000_3 --s 3 --kinds map_pass grad_pass lanczos_matvec > gpurun_out/passes_c4_final.jsonl 2>&1
timeout 300 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/prof_c4_final.jsonl 2>&1
timeout 300 python scripts/e2e_c4.py > gpurun_out/e2e_c4_final.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/bench_ncu_final.log 2>&1
bash scripts/ncu_pass.sh map_h23_sell H23 map_pass 2
exit 0
