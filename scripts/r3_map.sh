#!/bin/bash
# Round 2 (session 4): row-ordered SELL map pass for matrix completion.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_fullsize.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fullsize.log
timeout 300 python scripts/bench_passes.py mc400000_600000_3 --s 3 --kinds map_pass grad_pass lanczos_matvec > gpurun_out/passes_sellmap.jsonl 2>&1
CUHALLAR_NO_SELL_MAP=1 timeout 300 python scripts/bench_passes.py mc400000_600000_3 --s 3 --kinds map_pass > gpurun_out/passes_edgemap.jsonl 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_sellmap.json 2> gpurun_out/bench_sellmap.err
timeout 600 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/profile_c4_sellmap.jsonl 2>&1
bash scripts/ncu_pass.sh map_c4_sell C4 map_pass 3
exit 0
