#!/bin/bash
# One GPU call: bench line, ncu launch list, ncu --set full of the top kernels.
# usage: tools/profile_round.sh <scene>   (outputs under gpurun_out/)
set -x
SC=${1:-c5}
export PYTHONPATH=$PWD
mkdir -p gpurun_out
timeout 900 python bench.py --config $SC > gpurun_out/bench_$SC.json 2> gpurun_out/bench_$SC.err
# the captures start after the state preparation (--profile-from-start off;
# bench.py / prof_driver.py / one_step.py call cuProfilerStart)
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$SC.csv \
  python bench.py --config $SC --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_run.log 2>&1
for spec in "pcg:k_pcg33_stream:1" "spmv:k_spmv_sell:1" "asm:k_gather_h|k_grad_rows|k_block_rows:4" "eval:k_eval_stencil_b_tri:1" "evala:k_eval_stencil_a:1"; do
  IFS=: read tag rx cnt <<< "$spec"
  timeout 1200 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"$rx" -c $cnt \
    -f -o gpurun_out/prof_${tag}_$SC python tools/prof_driver.py $SC > gpurun_out/prof_driver_${tag}_$SC.log 2>&1
done
# FP64 work of the local evaluation (one Newton step: every k_eval* launch)
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum \
  --clock-control none -k regex:k_eval --csv --log-file gpurun_out/evalflops_$SC.csv python tools/one_step.py $SC 1 > gpurun_out/evalflops_run.log 2>&1
tail -3 gpurun_out/bench_$SC.err
cat gpurun_out/bench_$SC.json
