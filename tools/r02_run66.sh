mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
bash tools/prof_list.sh > gpurun_out/r02_list66.log 2>&1; head -50 gpurun_out/r02_list66.log; cp gpurun_out/launches_now.csv gpurun_out/launches_66.csv
for k in k_stream_match_ids k_rp_dec_cands; do
  timeout 900 bash tools/prof_kernel.sh $k 0 r02l_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02l_$k.ncu-rep 16 > gpurun_out/r02l_ncu_$k.txt 2>&1; head -30 gpurun_out/r02l_ncu_$k.txt
done
