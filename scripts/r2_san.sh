cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool initcheck python scripts/parity_aipp_once.py H12 > gpurun_out/initcheck_parity.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck python scripts/parity_aipp_once.py H12 > gpurun_out/racecheck_parity12.txt 2>&1
exit 0
