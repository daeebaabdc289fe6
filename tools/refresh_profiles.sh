#!/bin/bash
# GPU side of the profile refresh (run under gpurun): bench line, ncu launch
# list of the same command, ncu --set full of both batch kernels on the bench's
# 1M-module workload, and per-kernel times at 200k modules.  Outputs in
# gpurun_out/; tools/refresh_profiles.py copies / summarises them into profiles/.
cd "$(dirname "$0")/.."
python bench.py > gpurun_out/rp_bench.json 2> gpurun_out/rp_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/rp_launches.csv \
  python bench.py --steps 2 --warmup 3 > gpurun_out/rp_launch_bench.log 2>&1
for k in disasm asm; do
  ncu --set full --import-source on --clock-control none -k regex:^${k}_kernel -c 1 -o gpurun_out/rp_${k}_1M \
    python bench.py --steps 1 --warmup 3 > gpurun_out/rp_ncu_${k}.log 2>&1
done
for k in disasm asm validate; do python tools/prof_disasm.py --modules 200000 --kind $k; done > gpurun_out/rp_kernels_200k.txt 2>&1
tail -c 300 gpurun_out/rp_bench.json; cat gpurun_out/rp_kernels_200k.txt
