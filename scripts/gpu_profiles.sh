#!/bin/bash
# Round profiles (run under gpurun): the bench's ncu launch list, ncu --set full of the dominant GEMM
# (K=16384, 256x512 pair tile) next to cuBLAS, the hdim-128 attention kernel, the FP8 attention kernel
# and the hdim-64 causal kernel. Reports land in gpurun_out/.
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-vs-cublas > gpurun_out/bench_ncu_final.log 2>&1
K=16384 EXTRA="--bn 512" bash scripts/prof_gemm_vs_cublas.sh > /dev/null 2>&1
K=2048 bash scripts/prof_gemm_vs_cublas.sh > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_attn -s 1 -c 1 -o gpurun_out/prof_attn_final python scripts/prof_one.py attn > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_attn -s 1 -c 1 -o gpurun_out/prof_attn_fp8 python scripts/prof_one.py attn_fp8 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:ws_attn -s 1 -c 1 -o gpurun_out/prof_attn_c64 python scripts/prof_one.py attn_causal64 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep gpurun_out/launches_final.csv
# summaries (text) on the box; the .ncu-rep files exceed what gpurun copies back
python scripts/summarize_launches.py gpurun_out/launches_final.csv > gpurun_out/sum_launches.md
(echo "# ncu --set full, one launch each, bf16 8192x8192x16384: A = ours (256x512 cta_group::2 pair tile), B = cuBLAS nvjet"; \
 python scripts/ncu_cmp.py gpurun_out/prof_ours_k16384.ncu-rep gpurun_out/prof_cublas_k16384.ncu-rep; \
 python scripts/ncu_summary.py gpurun_out/prof_ours_k16384.ncu-rep --json gemm_bf16_8192x8192x16384) > gpurun_out/sum_gemm.txt 2>&1
(echo "# ncu --set full, one launch each, bf16 8192x8192x2048: A = ours (auto: 256x512 pair tile), B = cuBLAS nvjet"; \
 python scripts/ncu_cmp.py gpurun_out/prof_ours_k2048.ncu-rep gpurun_out/prof_cublas_k2048.ncu-rep; \
 python scripts/ncu_summary.py gpurun_out/prof_ours_k2048.ncu-rep --json gemm_bf16_8192x8192x2048) > gpurun_out/sum_gemm2048.txt 2>&1
for r in attn_final attn_fp8 attn_c64; do
  (python scripts/ncu_summary.py gpurun_out/prof_$r.ncu-rep --json $r; \
   ncu -i gpurun_out/prof_$r.ncu-rep --page source --csv --print-source sass > /tmp/src_$r.csv 2>/dev/null; \
   python scripts/ncu_stalls.py /tmp/src_$r.csv --top 20) > gpurun_out/sum_$r.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep gpurun_out/launches_final.csv
ls -la gpurun_out/sum_*
