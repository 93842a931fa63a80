#!/bin/bash
# Round-end evidence on one B200 (run under gpurun from the repo root):
# bench lines for every config + the reference arm, the cold launch list of
# the default bench, and `ncu --set full` captures of the hot kernels.
#   gpurun --timeout 3000 -- 'bash scripts/round_profile.sh r2'
set -u
R=${1:-r2}
O=gpurun_out/$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_papers100m.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_papers100m_reference.log 2>&1
for c in products oag cfg1; do
  timeout 900 python bench.py --config $c > $O/bench_$c.log 2>&1
done
# launch list (shares): ncu cannot replay kernel nodes of graphs with conditional
# nodes, so this pass runs with the size-switched GEMMs off (GNS_SWITCH_CHUNK=0)
GNS_SWITCH_CHUNK=0 ncu --metrics gpu__time_duration.sum --clock-control none -s 1500 -c 300 --csv \
    --log-file $O/launches_papers100m.csv \
    python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-extras --e2e-steps 0 > $O/ncu_launches.log 2>&1
# the timed configuration's training-branch HBM kernels, launched eagerly with the
# graph's arguments (switch on)
ncu --set full --clock-control none --import-source on --profile-from-start off -o $O/ncu_full_kernels \
    python scripts/kernel_ncu.py > $O/ncu_full_kernels.log 2>&1
# one sampling chain (3 layers + transposes)
ncu --set full --clock-control none --import-source on --profile-from-start off -o $O/ncu_full_sampler \
    python scripts/sampler_ncu.py > $O/ncu_full_sampler.log 2>&1
ls -la $O
