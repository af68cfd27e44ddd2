# One gpurun call that produces a round's evidence (writes gpurun_out/r2/).
set -x
O=gpurun_out/r2
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > $O/pytest_gpu.log 2>&1; echo rc=$? >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_cfg1.json 2> $O/bench_cfg1.err
timeout 600 python bench.py --workload cfg0 --no-cpu-baseline --steps 3000 > $O/bench_cfg0.json 2>&1
timeout 400 python bench.py --workload cfg2 --no-cpu-baseline > $O/bench_cfg2.json 2>&1
timeout 400 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2>&1
timeout 400 python bench.py --workload cfg3 --select kv_head --no-cpu-baseline > $O/bench_cfg3_kvhead.json 2>&1
for b in 1024 2048 4096 8192; do timeout 900 python bench.py --workload cfg4 --budget $b --no-cpu-baseline --steps 3 --e2e-steps 0 > $O/bench_cfg4_$b.json 2>&1; done
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
# serialised launch list of the default bench (share of each kernel)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"decode|merge|select|compact|fold" -c 800 --csv --log-file $O/launches_cfg1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu1.log 2>&1
# full captures of the top kernels (each command first runs plain)
python tools/probe.py --ncu > $O/plain_dec.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"decode_tcd_kernel|merge_kernel|select_kernel|compact_kernel|fold" -s 64 -c 6 -o $O/r2_dec_full python tools/probe.py --ncu > $O/ncu_dec.log 2>&1
REPS=1 python tools/probe_prefill.py > $O/plain_pf.log 2>&1 && \
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 -o $O/r2_prefill_full python tools/probe_prefill.py > $O/ncu_pf.log 2>&1
# config 3: the all-layer cluster kernel (one launch = 32 layers of a token) and its per-phase timeline
B=4096 timeout 120 python tools/probe_layers.py > $O/layers_cfg3.txt 2>&1 && \
B=4096 timeout 600 ncu --set full --import-source on --clock-control none -k regex:decode_tc_cluster -s 2 -c 1 -o $O/r2_cfg3_full python tools/probe_layers.py > $O/ncu_cfg3.log 2>&1
ls -la $O
