cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
(find / -path '*Eigen/Core' -not -path '/proc/*' 2>/dev/null | head -5; nproc; lscpu | grep -E 'Model name|^CPU\(s\)') > gpurun_out/eigen_probe.txt
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python scripts/parity_compare.py C5 petersen H4 H6 H8 H10 mc30 mc100 H12 mc2000 H13 H14 > gpurun_out/parity_cmp.jsonl 2> gpurun_out/parity_cmp.err
exit 0
