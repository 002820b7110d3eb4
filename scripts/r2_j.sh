cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/sell_ab.py C4 H23 H20 > gpurun_out/sell_ab3.jsonl 2> gpurun_out/sell_ab3.err
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/profile_c4b.jsonl 2>&1
exit 0
