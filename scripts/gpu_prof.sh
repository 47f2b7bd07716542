# source-level profile of one small batched launch of the C4 tile kernel
python scripts/prof_c4.py 1184 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:lse_reg --launch-skip 4 -c 1 -o gpurun_out/prof_c4c python scripts/prof_c4.py 1184 > gpurun_out/ncu.log 2>&1
echo rc=$?
tail -2 gpurun_out/ncu.log
