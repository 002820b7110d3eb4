cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/sell_ab.py C4 H23 > gpurun_out/sell_ab6.jsonl 2> gpurun_out/sell_ab6.err
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_tma.log 2>&1
exit 0
