python scripts/run_big.py --config C3 --scale 4 --oracle > gpurun_out/c3q.json 2> gpurun_out/c3q.err; echo rc=$?; cat gpurun_out/c3q.json; tail -3 gpurun_out/c3q.err
python scripts/run_big.py --config C3 > gpurun_out/c3.json 2> gpurun_out/c3.err; echo rc=$?; cat gpurun_out/c3.json; tail -3 gpurun_out/c3.err
python scripts/run_big.py --config C5 --scale 4 --oracle > gpurun_out/c5q.json 2> gpurun_out/c5q.err; echo rc=$?; cat gpurun_out/c5q.json; tail -3 gpurun_out/c5q.err
python scripts/run_big.py --config C5 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo rc=$?; cat gpurun_out/c5.json; tail -3 gpurun_out/c5.err
