#!/bin/bash
# H(23,2) with a 300 s solver time limit: does the certificate already meet 1e-5?
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python scripts/solve_large.py H23 --time-limit 300 --profile > gpurun_out/c5_limit300.jsonl 2> gpurun_out/c5_limit300.err
exit 0
