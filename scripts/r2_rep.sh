cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 300 python scripts/parity_repeat.py H10 8 > gpurun_out/rep.txt 2>&1
timeout 300 python scripts/parity_repeat.py H8 8 >> gpurun_out/rep.txt 2>&1
timeout 300 python scripts/parity_repeat.py H12 3 >> gpurun_out/rep.txt 2>&1
cat > /tmp/h4.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2505_13719_b200 as H
inst = H.build_theta_instance(H.make_hypercube(4))
r = H.solve(inst, H.SolverConfig(eps=1e-5, seed=0, parity=True))
print(r.fista_iters)
PY
timeout 600 compute-sanitizer --tool racecheck python /tmp/h4.py > gpurun_out/racecheck_parity.txt 2>&1
timeout 600 compute-sanitizer --tool synccheck python /tmp/h4.py > gpurun_out/synccheck_parity.txt 2>&1
exit 0
