cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gauss_pr.py -q -x > gpurun_out/pytest_gauss.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/sell_ab.py C4 H23 > gpurun_out/sell_ab7.jsonl 2> gpurun_out/sell_ab7.err
timeout 600 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/profile_c4e.jsonl 2>&1
exit 0
