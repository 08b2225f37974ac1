# ncu evidence for the N=1 bench (C2): launch list + one full capture of the put kernel.
# --no-overlap: ncu serialises kernels, so the next put must not wait on a concurrent consume.
set -e
python bench.py --steps 20 --warmup 3 --cpu-budget 0.2 --no-overlap > gpurun_out/plain_c2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c2.csv \
    python bench.py --steps 20 --warmup 3 --cpu-budget 0.2 --no-overlap > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:put_kernel -s 10 -c 1 -o gpurun_out/prof_put_c2 \
    python bench.py --steps 20 --warmup 3 --cpu-budget 0.2 --no-overlap > gpurun_out/ncu_full.log 2>&1
python tools/ncu_summary.py list gpurun_out/launches_c2.csv gpurun_out/ncu_launches_c2.json > /dev/null
python tools/ncu_summary.py rep gpurun_out/prof_put_c2.ncu-rep gpurun_out/ncu_put_c2.json > /dev/null
echo prof_done
