cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
# old (round-1) library vs the current one on the operator path
(cd scratch_old && timeout 300 python ../scripts/repro_map.py 10 16 > ../gpurun_out/repro_old.txt 2>&1)
timeout 300 python scripts/repro_map.py 10 16 > gpurun_out/repro_new.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_devgen.py -q -x > gpurun_out/pytest_devgen.log 2>&1
timeout 600 python - > gpurun_out/gen_times.txt 2>&1 <<'PY'
import time, sys
sys.path.insert(0, '.')
import paper_2505_13719_b200 as H
for spec in [H.McSpec(400000, 600000, 3, 0), H.McSpec(3200000, 4800000, 3, 0, draws_per_dim=40)]:
    t = time.perf_counter(); i = H.gen_matrix_completion(spec); print(spec, i.m, time.perf_counter() - t, flush=True); del i
t = time.perf_counter(); i = H.build_theta_instance(H.make_hypercube(23)); print("H23", i.m, time.perf_counter() - t, flush=True)
PY
exit 0
