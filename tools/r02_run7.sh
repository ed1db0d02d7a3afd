# bench with REPLAY in the step; launch list; compute-sanitizer; ncu full captures of the top kernels
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python bench.py --cpu-budget 2 > gpurun_out/r02_bench7.json 2> gpurun_out/r02_bench7.err; echo "bench rc=$?"; head -c 2500 gpurun_out/r02_bench7.json; tail -5 gpurun_out/r02_bench7.err
python tools/sanitize.py > gpurun_out/r02_sanitize_plain.log 2>&1; echo "sanitize plain rc=$?"; tail -3 gpurun_out/r02_sanitize_plain.log
for tool in memcheck synccheck racecheck; do
  for w in c1 c2 c4; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize.py $w > gpurun_out/r02_sanitize_${tool}_$w.log 2>&1
    echo "$tool $w rc=$?"; tail -2 gpurun_out/r02_sanitize_${tool}_$w.log
  done
done
bash tools/prof_list.sh > gpurun_out/r02_list.log 2>&1; cat gpurun_out/r02_list.log | head -45
for k in k_window_sa k_stream_match k_stream_emit k_seg_sort1; do
  timeout 600 bash tools/prof_kernel.sh $k 0 r02_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02_$k.ncu-rep 20 > gpurun_out/r02_ncu_$k.txt 2>&1; head -40 gpurun_out/r02_ncu_$k.txt
done
