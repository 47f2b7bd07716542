mkdir -p gpurun_out
timeout 300 python scripts/wy_bench.py 2>&1 | grep -E "NT|TN|NN" 
echo "--- NT at BK=32"
MLSB_GEMM_NT32=1 timeout 300 python scripts/wy_bench.py 2>&1 | grep -E "NT"
echo "--- all at BK=16"
MLSB_GEMM_BK16=1 timeout 300 python scripts/wy_bench.py 2>&1 | grep -E "NT|TN|NN"
