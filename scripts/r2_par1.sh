cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python scripts/parity_compare.py C5 petersen H4 H6 mc30 mc100 H8 H10 H12 > gpurun_out/parity1.jsonl 2> gpurun_out/parity1.err
exit 0
