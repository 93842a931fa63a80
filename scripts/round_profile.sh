#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
# bench lines for every config + the reference arm, the cold launch list of
# the default bench, and one `ncu --set full` capture of the hot kernels.
#   gpurun --timeout 3000 -- 'bash scripts/round_profile.sh r1'
set -u
R=${1:-r1}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py > $O/bench_papers100m.log 2>&1
timeout 600 python bench.py --impl reference > $O/bench_papers100m_reference.log 2>&1
for c in products oag cfg1; do
  timeout 600 python bench.py --config $c > $O/bench_$c.log 2>&1
done
# ncu cannot profile kernel nodes of graphs with conditional nodes: profile with the
# size-switched GEMMs off (GNS_SWITCH_CHUNK=0; every other kernel is identical)
export GNS_SWITCH_CHUNK=0
ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 300 --csv --log-file $O/launches_papers100m.csv \
    python bench.py --steps 20 --warmup 10 --no-cpu-baseline --e2e-steps 0 > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"spmm_fwd_narrow|spmm_bwd_kernel|spmm_fwd_kernel" \
    -s 6 -c 5 -o $O/ncu_full_step python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_full_step.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sample_warp|sample_stream|layer_count_reduce|enumerate_apply" \
    -s 24 -c 8 -o $O/ncu_full_sampler python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_full_sampler.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"gather_f32x4" -s 2 -c 2 -o $O/ncu_full_gather \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $O/ncu_full_gather.log 2>&1
ls -la $O
