mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
bash tools/prof_list.sh > gpurun_out/r02_list59.log 2>&1; head -45 gpurun_out/r02_list59.log; cp gpurun_out/launches_now.csv gpurun_out/launches_59.csv
for k in k_stream_ends; do
  timeout 900 bash tools/prof_kernel.sh $k 0 r02i_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02i_$k.ncu-rep 16 > gpurun_out/r02i_ncu_$k.txt 2>&1; head -45 gpurun_out/r02i_ncu_$k.txt
done
