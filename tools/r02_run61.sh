mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for k in k_window_select; do
  timeout 900 bash tools/prof_kernel.sh $k 0 r02j_$k > /dev/null 2>&1; python tools/ncu_report.py gpurun_out/prof_r02j_$k.ncu-rep 25 > gpurun_out/r02j_ncu_$k.txt 2>&1; head -60 gpurun_out/r02j_ncu_$k.txt
done
