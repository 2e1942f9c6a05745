#!/bin/bash
# ncu counters for every feasible dp_sweep config (one launch each, after 2 warm-up launches):
# tensor-pipe activity, DRAM bytes and time, and warp-state samples per SASS instruction (the
# mbarrier-wait share is read from the SYNCS instructions by scripts/dp_sweep_report.py, on the box:
# only the JSON rows come back).
mkdir -p gpurun_out/dp
for c in $(python scripts/dp_sweep.py --list --ncu-subset); do
  timeout 300 ncu --clock-control none --import-source on \
    --section SpeedOfLight --section MemoryWorkloadAnalysis --section WarpStateStats --section SourceCounters \
    --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second \
    -k regex:ws_ -s 2 -c 1 -o /tmp/dp_$c -f python scripts/dp_sweep.py --one $c > /tmp/dp_$c.log 2>&1
  if [ -f /tmp/dp_$c.ncu-rep ]; then
    python scripts/dp_sweep_report.py /tmp/dp_$c.ncu-rep >> gpurun_out/dp/rows.jsonl
    rm -f /tmp/dp_$c.ncu-rep
  else
    echo "{\"id\": \"$c\", \"status\": \"no report\"}" >> gpurun_out/dp/rows.jsonl
    tail -3 /tmp/dp_$c.log >> gpurun_out/dp/errors.log
  fi
done
wc -l gpurun_out/dp/rows.jsonl
