set -x
timeout 1500 python -m pytest tests -m gpu -q --durations=12 > gpurun_out/r02_gputest.log 2>&1; echo "pytest_rc=$?" >> gpurun_out/r02_gputest.log
tail -3 gpurun_out/r02_gputest.log
bash tools/ncu_r02.sh
python __graft_entry__.py > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo bench_rc=$?
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo ref_rc=$?
timeout 600 python bench.py --config 1 --extra "" --schedule random --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_c1_random.json 2>/dev/null
timeout 600 python bench.py --config 3 --extra "2" --schedule random --no-e2e --no-cpu-baseline > gpurun_out/r02_bench_c3_random.json 2>/dev/null
ls -la gpurun_out
