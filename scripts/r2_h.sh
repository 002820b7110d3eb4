cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/sell_ab.py C4 H23 H20 > gpurun_out/sell_ab.jsonl 2> gpurun_out/sell_ab.err
timeout 1800 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
exit 0
