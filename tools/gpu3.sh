mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 2 --cpu-budget 3 > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench rc=$?"; cat gpurun_out/bench3.json; tail -5 gpurun_out/bench3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench3_ref.json 2>&1; echo "ref rc=$?"; cat gpurun_out/bench3_ref.json
timeout 600 python bench.py --config C3 --steps 5 --warmup 3 --cpu-budget 3 > gpurun_out/bench3_c3.json 2> gpurun_out/bench3_c3.err; echo "c3 rc=$?"; cat gpurun_out/bench3_c3.json; tail -3 gpurun_out/bench3_c3.err
