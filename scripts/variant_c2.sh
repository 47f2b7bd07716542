# A/B timing of prebuilt library variants (variants/*.so) on the C2 stamps
mkdir -p gpurun_out
cp paper_2406_16499_b200/lib/libmixedls_b200.so /tmp/cur.so
for v in variants/*.so; do
  cp $v paper_2406_16499_b200/lib/libmixedls_b200.so
  echo "== $v" >> gpurun_out/variants.log
  MLSB_DEBUG_STAMPS=1 timeout 300 python scripts/c2_stamps.py >> gpurun_out/variants.log 2>&1
done
cp /tmp/cur.so paper_2406_16499_b200/lib/libmixedls_b200.so
