# Round-end GPU evidence: GPU tests, bench line (config 4 headline), all-config table, ncu launch list of
# the timed region and --set full captures of the top kernels.  usage: bash tools/gpu_round.sh <tag>
set -x
T=${1:-r02}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 1200 python bench.py > gpurun_out/bench_$T.jsonl 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --config 1 --no-configs --no-cpu-baseline > gpurun_out/bench1_$T.jsonl 2> gpurun_out/bench1_$T.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.jsonl 2> gpurun_out/bench_ref_$T.err
timeout 900 python tools/run_configs.py > gpurun_out/configs_$T.jsonl 2> gpurun_out/configs_$T.err
FI_GMRES_DEVICE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_l_$T.log 2>&1
FI_GMRES_DEVICE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:tau_pcg_fused --launch-skip 1 -c 1 --profile-from-start off -f -o gpurun_out/prof_k5_$T python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_k5_$T.log 2>&1
FI_GMRES_DEVICE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:toeplitz_apply -c 1 --profile-from-start off -f -o gpurun_out/prof_k1_$T python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_k1_$T.log 2>&1
FI_GMRES_DEVICE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:mgs_step -c 1 --profile-from-start off -f -o gpurun_out/prof_k3_$T python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_k3_$T.log 2>&1
FI_GMRES_DEVICE=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:hodlr_sweep -c 1 --profile-from-start off -f -o gpurun_out/prof_k2h_$T python bench.py --config 1 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_k2h_$T.log 2>&1
FI_GMRES_DEVICE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches1_$T.csv python bench.py --config 1 --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_l1_$T.log 2>&1
tail -3 gpurun_out/pytest_gpu_$T.log; cat gpurun_out/bench_$T.jsonl
