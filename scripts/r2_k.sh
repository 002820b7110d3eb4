cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 600 python scripts/sell_ab.py C4 H23 > gpurun_out/sell_ab4.jsonl 2> gpurun_out/sell_ab4.err
timeout 600 python scripts/profile_solve.py mc400000_600000_3 > gpurun_out/profile_c4c.jsonl 2>&1
exit 0
