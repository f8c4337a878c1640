#!/bin/bash
# One GPU session: smoke, tests, bench, ncu launch list of one solve + full capture of the
# fine Jacobi sweep (k_stream<JacobiOp>).   usage: tools/gpu_round.sh TAG [skip-tests]
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_solve.py > gpurun_out/launches_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off \
   -k regex:k_stream -s 2 -c 1 -o gpurun_out/jacobi_$TAG -f python tools/profile_kernel.py --kernels jacobi \
   > gpurun_out/ncu_full_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --profile-from-start off \
   -k regex:k_stream -s 2 -c 1 -o gpurun_out/uzawa_$TAG -f python tools/profile_kernel.py --kernels pupdate \
   > gpurun_out/ncu_uzawa_$TAG.log 2>&1
ls -la gpurun_out
