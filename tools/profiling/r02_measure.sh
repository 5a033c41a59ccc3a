#!/bin/bash
# Round-2 measurement set (B200, one GPU): the default bench line, the other BASELINE workloads, the dS-path
# variant, the ncu launch list of the bench command and one ncu --set full capture of the top kernels.
# Outputs under gpurun_out/r02/ (copied to profiles/ by hand).
set -u
O=gpurun_out/r02; mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_32k.json 2> $O/bench_32k.err
python bench.py --config wan14b_75k --steps 5 --warmup 3 --dense-steps 1 --no-cpu-baseline > $O/bench_75k.json 2> $O/bench_75k.err
python bench.py --config long_147k --steps 3 --warmup 3 --dense-steps 0 --no-cpu-baseline > $O/bench_147k.json 2> $O/bench_147k.err
BSA_BWD_PATH=ds python tools/profiling/time_attn.py wan1.3b_32k 20 > $O/time_ds_32k.txt 2>&1
python tools/profiling/time_attn.py wan1.3b_32k 20 > $O/time_reduce_32k.txt 2>&1
BSA_BWD_PATH=ds python tools/profiling/time_attn.py wan14b_75k 5 > $O/time_ds_75k.txt 2>&1
python tools/profiling/time_attn.py wan14b_75k 5 > $O/time_reduce_75k.txt 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --dense-steps 0 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"k_attn_bwd|k_attn_fwd|k_select_queries|k_scores|k_admit|k_bwd_prep|k_kv_image|k_pool|k_bwd_finalize|k_fill" \
  -c 12 -o $O/prof_full python tools/profiling/time_attn.py wan1.3b_32k 1 > $O/ncu_full.log 2>&1
