# ncu captures for profiles/ (one gpurun call; each command first runs plain)
set -x
python tools/probe.py --ncu > gpurun_out/plain_dec.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"decode_kernel|merge_kernel|select_kernel|compact_kernel|fold" -s 64 -c 6 -o gpurun_out/r1_dec_full python tools/probe.py --ncu > gpurun_out/ncu_dec.log 2>&1
REPS=1 python tools/probe_prefill.py > gpurun_out/plain_pf.log 2>&1 && \
REPS=1 ncu --set full --clock-control none --import-source on -k regex:prefill_kernel -s 2 -c 1 -o gpurun_out/r1_prefill_full python tools/probe_prefill.py > gpurun_out/ncu_pf.log 2>&1
python tools/probe_chunk.py > gpurun_out/plain_chunk.log 2>&1 && \
ncu --set full --clock-control none -k regex:"fold_rows|append_chunk" -c 2 -o gpurun_out/r1_chunk_full python tools/probe_chunk.py > gpurun_out/ncu_chunk.log 2>&1
S=1 HKV=8 B=4096 E=256 STEPS=6 RECORD=0 python tools/probe_decode.py > gpurun_out/plain_cfg3.log 2>&1 && \
S=1 HKV=8 B=4096 E=256 STEPS=6 RECORD=0 ncu --set full --clock-control none -k regex:"decode_tc_kernel|merge_kernel" -s 12 -c 2 -o gpurun_out/r1_cfg3_full python tools/probe_decode.py > gpurun_out/ncu_cfg3.log 2>&1
ls -la gpurun_out/*.ncu-rep
