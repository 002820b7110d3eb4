cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_refill.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_refill.log 2>&1
timeout 600 python scripts/sell_ab.py C4 H23 > gpurun_out/sell_ab2.jsonl 2> gpurun_out/sell_ab2.err
timeout 600 python scripts/profile_solve.py mc400000_600000_3 H16 > gpurun_out/profile_c4.jsonl 2>&1
bash scripts/ncu_pass.sh c4_grad_sell C4 grad_pass 3
bash scripts/ncu_pass.sh h23_grad_sell H23 grad_pass 2
CUHALLAR_NO_SELL=1 bash scripts/ncu_pass.sh h23_grad_rt H23 grad_pass 2
bash scripts/ncu_pass.sh c4_map C4 map_pass 3
du -sh gpurun_out
exit 0
