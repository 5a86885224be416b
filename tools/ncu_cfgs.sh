#!/bin/bash
export HARRIS_DEV=1  # developer knobs (HARRIS_*_CONFIG, HARRIS_BAND_ROWS, ...) are read only with this
# dev: focused ncu metrics for several TMA configs on the batch workload (1 launch each)
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__inst_executed.sum,sm__cycles_elapsed.avg.per_second,dram__throughput.avg.pct_of_peak_sustained_elapsed
for c in ${CFGS:-0 1 6}; do
  mkdir -p gpurun_out
  HARRIS_TMA_CONFIG=$c timeout 300 ncu --metrics $M --clock-control none -k regex:strip_kernel -s 3 -c 1 --csv --log-file gpurun_out/ncu_cfg$c.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-extra --no-cpu-baseline > /dev/null 2>&1
  python -c "
import csv,sys
rows=[r for r in csv.reader(open('gpurun_out/ncu_cfg$c.csv')) if len(r) > 10]
h=rows[0]; mi=h.index('Metric Name'); vi=h.index('Metric Value')
out={r[mi].replace('smsp__average_warps_issue_stalled_','st_').replace('_per_issue_active.ratio',''):r[vi] for r in rows[1:] if len(r)>vi}
print('cfg$c', out)"
done
