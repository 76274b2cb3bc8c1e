set -x
T=${1:-r02f}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$T.log
timeout 1200 python bench.py > gpurun_out/bench_$T.jsonl 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.jsonl 2> gpurun_out/bench_ref_$T.err
timeout 900 python bench.py --config 1 --no-configs --no-cpu-baseline > gpurun_out/bench1_$T.jsonl 2> gpurun_out/bench1_$T.err
FI_GMRES_DEVICE=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline --no-configs > gpurun_out/ncu_l_$T.log 2>&1
tail -3 gpurun_out/pytest_gpu_$T.log; cat gpurun_out/bench_$T.jsonl | head -c 3000
