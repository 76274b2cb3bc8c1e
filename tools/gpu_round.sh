set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_r01f.jsonl 2> gpurun_out/bench_r01f.err
timeout 900 python tools/run_configs.py > gpurun_out/configs_r01f.jsonl 2> gpurun_out/configs_r01f.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hodlr_sweep -c 1 --profile-from-start off -f -o gpurun_out/prof_k2h_r01f python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:toeplitz_apply -c 1 --profile-from-start off -f -o gpurun_out/prof_k1_r01f python bench.py --steps 1 --warmup 3 --profile --no-cpu-baseline > gpurun_out/ncu_f1.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_r01f.jsonl
