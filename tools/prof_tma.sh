# ncu evidence for the TMA engine over NVLink (2-GPU box): the put of 32 x 4 MiB into a
# peer ring by the LSU copy warps (33 CTAs x 512) and by the TMA engine (17 and 33 CTAs,
# 6 engine warps each): duration, NVLink bytes, instructions issued, SM throughput.
set -e
M=gpu__time_duration.sum,nvltx__bytes.sum,nvltx__bytes_data_user.sum,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size
for cfg in 33:512:0 17:0:1 33:0:1; do
  PUT_CFG=$cfg python tools/ncu_targets.py nvlink > /dev/null
  PUT_CFG=$cfg ncu --metrics $M --clock-control none -k regex:put_kernel -s 2 -c 3 --csv \
      --log-file gpurun_out/r02b_ncu_tma_$cfg.csv python tools/ncu_targets.py nvlink > /dev/null 2>&1
done
echo prof_tma_done
