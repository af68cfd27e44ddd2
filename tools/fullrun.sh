set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_cfg1.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 300 python bench.py --workload cfg0 --no-cpu-baseline > gpurun_out/bench_cfg0.log 2>&1
timeout 400 python bench.py --workload cfg2 --no-cpu-baseline > gpurun_out/bench_cfg2.log 2>&1
timeout 400 python bench.py --workload cfg3 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1
for b in 1024 2048 4096 8192; do timeout 900 python bench.py --workload cfg4 --budget $b --no-cpu-baseline --steps 3 --e2e-steps 0 > gpurun_out/bench_cfg4_$b.log 2>&1; done
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode_kernel|merge_kernel|select_kernel|compact_kernel|fold" -c 600 --csv --log-file gpurun_out/launches_cfg1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu1.log 2>&1
