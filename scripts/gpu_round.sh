#!/bin/bash
# Round-end style GPU pass: parity suite, bench line (+ reference arm), launch list,
# ncu captures of the dominant pass at the headline and north-star sizes.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-large > gpurun_out/bench_ncu.log 2>&1
bash scripts/ncu_capture.sh grad_H12 H12 grad_pass 2 400
bash scripts/ncu_capture.sh grad_H23 H23 grad_pass 2 3
exit 0
