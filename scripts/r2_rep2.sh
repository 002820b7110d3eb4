cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python scripts/parity_repeat.py H12 4 > gpurun_out/rep2.txt 2>&1
timeout 900 compute-sanitizer --tool initcheck python scripts/parity_aipp_once.py H12 > gpurun_out/initcheck_parity.txt 2>&1
timeout 900 python scripts/parity_compare.py mc300 mc1000 mc2000 H11 >> gpurun_out/rep2.txt 2>&1
exit 0
