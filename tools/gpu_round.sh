#!/bin/bash
# One GPU session: smoke, tests, bench, ncu launch list of one solve + full captures of the
# fine-level hot kernels (two-sweep pass = dominant, single sweep, fused Uzawa step,
# residual+restriction) at 4096^2; with "extra": also the RBGS passes, residual+energy, the
# fine kernels at 2048^2 and the GCR fused passes.   usage: tools/gpu_round.sh TAG [skip-tests] [extra]
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1
fi
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
   --log-file gpurun_out/launches_$TAG.csv python tools/profile_solve.py > gpurun_out/launches_$TAG.log 2>&1
N="ncu --set full --clock-control none --import-source on --profile-from-start off"
for K in jacobi2:k_jacobi2 jacobi:k_stream jacobi_uzawa:k_stream_bar residual_restrict:k_resrestrict; do
  timeout 900 $N -k regex:${K#*:} -s 2 -c 1 -o gpurun_out/${K%%:*}_$TAG -f python tools/profile_kernel.py --kernels ${K%%:*} \
     > gpurun_out/ncu_${K%%:*}_$TAG.log 2>&1
done
if [ "$3" == "extra" ]; then
  timeout 600 $N -k regex:k_rbgs_pass -c 2 -o gpurun_out/rbgs_4096_$TAG -f python tools/profile_kernel.py --kernels rbgs > /dev/null 2>&1
  timeout 600 $N -k regex:k_stream -c 1 -o gpurun_out/energy_4096_$TAG -f python tools/profile_kernel.py --kernels energy > /dev/null 2>&1
  for K in jacobi2:k_jacobi2 jacobi:k_stream jacobi_uzawa:k_stream_bar residual_restrict:k_resrestrict prolong:k_prolong2; do
    timeout 600 $N -k regex:${K#*:} -s 2 -c 1 -o gpurun_out/${K%%:*}_2048_$TAG -f python tools/profile_kernel.py --n 2048 --kernels ${K%%:*} > /dev/null 2>&1
  done
  timeout 900 $N -k regex:"k_mgs_step|k_gcr_update|k_gcr_final" -c 8 -o gpurun_out/gcr_solcx2048_$TAG -f \
     python tools/profile_solve.py --workload solcx --max-iter 3 > /dev/null 2>&1
fi
ls -la gpurun_out
