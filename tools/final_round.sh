#!/bin/bash
# Round-end evidence on one B200: smoke, the whole GPU suite, the bench line, the ncu launch list
# of one solve (serialised, cold cache; share of the step per kernel).   usage: tools/final_round.sh TAG
TAG=${1:-r02u}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc $?" >> gpurun_out/bench_$TAG.err
timeout 900 python tools/profile_solve.py > /dev/null 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_solve.py > gpurun_out/launches_$TAG.log 2>&1
tail -2 gpurun_out/smoke_$TAG.log; tail -3 gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/bench_$TAG.json; tail -2 gpurun_out/bench_$TAG.err
