#!/bin/bash
# One GPU-box round trip: parity tests, bench line, launch list, pass timings, ncu capture.
set -x
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 900 python scripts/bench_passes.py ${PASS_INSTANCES:-H12 H20 H23 mc2000_2000_3} --s 1 2 3 > gpurun_out/passes.jsonl 2> gpurun_out/passes.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hallar -s 1 -c 1 -o gpurun_out/prof_grad_H20 python scripts/ncu_pass.py H20 grad_pass 2 5 > gpurun_out/ncu_full.log 2>&1
exit 0
