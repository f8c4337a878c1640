#!/bin/bash
# One GPU session: tests, bench, ncu launch list + full capture of the Jacobi sweep.
# usage: tools/gpu_round.sh TAG [skip-tests]
set -x
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_$TAG.log 2>&1
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_solve.py > gpurun_out/launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:k_jacobi -s 20 -c 1 -o gpurun_out/jacobi_$TAG -f python tools/profile_solve.py --max-iter 3 > gpurun_out/ncu_full_$TAG.log 2>&1
ls -la gpurun_out
