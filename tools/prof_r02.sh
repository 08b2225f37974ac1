# ncu evidence, round 2 (run on a 2-GPU box under gpurun; each command first runs clean without ncu):
#   C2 launch list + full put capture (prof_c2.sh), copy-out get, NVLink put / get with nvltx / nvlrx bytes.
set -e
mkdir -p gpurun_out
NVL=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/ncu_targets.py nvlink
python tools/ncu_targets.py copyout
bash tools/prof_c2.sh
ncu --metrics $NVL --clock-control none -k regex:"put_kernel|get_kernel" --csv --log-file gpurun_out/r02_ncu_nvlink_counters.csv \
    python tools/ncu_targets.py nvlink > gpurun_out/r02_ncu_nvlink_counters.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:put_kernel -s 3 -c 1 -o gpurun_out/r02_prof_put_nvlink \
    python tools/ncu_targets.py nvlink > gpurun_out/r02_ncu_put_nvlink.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:get_kernel -c 1 -o gpurun_out/r02_prof_get_nvlink \
    python tools/ncu_targets.py nvlink > gpurun_out/r02_ncu_get_nvlink.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:get_kernel -s 1 -c 1 -o gpurun_out/r02_prof_get_copyout \
    python tools/ncu_targets.py copyout > gpurun_out/r02_ncu_get_copyout.log 2>&1
python tools/ncu_summary.py rep gpurun_out/r02_prof_put_nvlink.ncu-rep gpurun_out/r02_ncu_put_nvlink.json > /dev/null
python tools/ncu_summary.py rep gpurun_out/r02_prof_get_nvlink.ncu-rep gpurun_out/r02_ncu_get_nvlink.json > /dev/null
python tools/ncu_summary.py rep gpurun_out/r02_prof_get_copyout.ncu-rep gpurun_out/r02_ncu_get_copyout.json > /dev/null
echo prof_r02_done
