cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
find / -path '*Eigen/Core' -not -path '/proc/*' 2>/dev/null | head -5 > gpurun_out/eigen_probe.txt
nproc >> gpurun_out/eigen_probe.txt; lscpu | grep -E 'Model name|^CPU\(s\)' >> gpurun_out/eigen_probe.txt
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
exit 0
