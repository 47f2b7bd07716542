# harness cells (routed vs plain reference), FFMA issue-form rates, C4 stage stamps
mkdir -p gpurun_out
MIXEDLS_THREADS=1 timeout 600 oracle/_ref/b200_harness lse > gpurun_out/harn_gpu_lse.txt 2>&1; echo harn_gpu=$?
MIXEDLS_THREADS=16 timeout 600 oracle/_ref/ref_harness lse > gpurun_out/harn_ref_lse.txt 2>&1; echo harn_ref=$?
timeout 120 scripts/micro/ffma_rates > gpurun_out/ffma_rates.txt 2>&1; cat gpurun_out/ffma_rates.txt
MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/prof_c4.py 1184 > gpurun_out/stamps_c4.txt 2>&1; grep -E "STAMPS|phases|batch" gpurun_out/stamps_c4.txt | tail -4
