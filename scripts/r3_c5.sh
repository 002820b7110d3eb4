#!/bin/bash
# North-star H(23,2) solve to 1e-5 with the final build (row-ordered theta map), per-phase profile.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2700 python scripts/solve_large.py H23 --time-limit 2500 --profile > gpurun_out/c5_final.jsonl 2> gpurun_out/c5_final.err
exit 0
