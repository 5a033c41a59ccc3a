#!/bin/bash
# Round-2 closing measurement set (one B200): the GPU test suite with the parity record, the bench lines of the
# BASELINE workloads, the ncu launch list of the bench command, one ncu --set full capture of the step's kernels
# and the anneal run. Outputs under gpurun_out/final/.
set -u
O=gpurun_out/final; mkdir -p $O
BSA_PARITY_OUT=$O/r02_parity.json timeout 1500 python -m pytest tests -m gpu -q > $O/gputests.txt 2>&1; echo "exit $?" >> $O/gputests.txt
python bench.py --steps 20 --warmup 5 > $O/bench_32k.json 2> $O/bench_32k.err
python bench.py --config wan14b_75k --steps 5 --warmup 3 --dense-steps 1 --no-cpu-baseline > $O/bench_75k.json 2> $O/bench_75k.err
python bench.py --config long_147k --steps 3 --warmup 3 --dense-steps 0 --no-cpu-baseline > $O/bench_147k.json 2> $O/bench_147k.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
python tools/training/anneal_run.py --steps 1000 --out $O/r02_anneal.json > $O/anneal.log 2>&1
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --dense-steps 0 --e2e-steps 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on \
  -k regex:"k_attn_bwd|k_attn_fwd|k_select_queries|k_scores|k_admit|k_bwd_prep|k_kv_image|k_pool|k_bwd_finalize|k_fill|k_k2q|k_partition" \
  -c 14 -o $O/prof_full python tools/profiling/time_attn.py wan1.3b_32k 1 > $O/ncu_full.log 2>&1
