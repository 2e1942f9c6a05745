#!/bin/bash
# One GPU session: tests, smoke, bench, launch list, ncu full captures. Outputs in gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ws_gemm -s 2 -c 1 -o gpurun_out/prof_gemm_k16384 python scripts/prof_one.py gemm --K 16384 --cta_pair > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ws_attn -s 1 -c 1 -o gpurun_out/prof_attn python scripts/prof_one.py attn > gpurun_out/ncu_attn.log 2>&1
ls -la gpurun_out
