mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
bash tools/prof_list.sh > gpurun_out/r02_list50.log 2>&1; head -30 gpurun_out/r02_list50.log; cp gpurun_out/launches_now.csv gpurun_out/launches_50.csv
for k in k_stream_match_ids k_stream_emit; do
  timeout 900 bash tools/prof_kernel.sh $k 0 r02h_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02h_$k.ncu-rep 16 > gpurun_out/r02h_ncu_$k.txt 2>&1; head -45 gpurun_out/r02h_ncu_$k.txt
done
