#!/bin/bash
# Final round pass: parity suite, bench line (+ reference arm), launch list, and the
# north-star matrix-completion instances with the paper's sampling rule.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-large > gpurun_out/bench_ncu.log 2>&1
timeout 1500 python scripts/solve_large.py mcp400000_600000_3 mcp3200000_4800000_3 --time-limit 900 --profile \
  > gpurun_out/large_mcp.jsonl 2> gpurun_out/large_mcp.err
exit 0
