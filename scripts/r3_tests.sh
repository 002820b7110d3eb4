#!/bin/bash
# Final GPU suite of the committed tree + smoke().
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_last.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_last.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_last.log 2>&1; echo "rc=$?" >> gpurun_out/smoke_last.log
exit 0
