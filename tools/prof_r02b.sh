# ncu evidence, round 2 part b (2-GPU box; each target first runs clean without ncu):
#   C2 launch list + full put capture (prof_c2.sh) after the ragged-tail change, and the split-placement
#   copy-out consume (get_kernel<true> pulling over NVLink) with NVLink counters and one full capture.
set -e
mkdir -p gpurun_out
NVL=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,nvltx__bytes_data_protocol.sum,nvlrx__bytes.sum,nvlrx__bytes_data_user.sum,nvlrx__bytes_data_protocol.sum,dram__bytes_read.sum,dram__bytes_write.sum
python tools/ncu_targets.py split
bash tools/prof_c2.sh
ncu --metrics $NVL --clock-control none -k regex:"put_kernel|get_kernel" --csv --log-file gpurun_out/r02b_ncu_split_counters.csv \
    python tools/ncu_targets.py split > gpurun_out/r02b_ncu_split_counters.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:get_kernel -s 2 -c 1 -o gpurun_out/r02b_prof_get_split \
    python tools/ncu_targets.py split > gpurun_out/r02b_ncu_get_split.log 2>&1
python tools/ncu_summary.py rep gpurun_out/r02b_prof_get_split.ncu-rep gpurun_out/r02b_ncu_get_split.json > /dev/null
echo prof_r02b_done
