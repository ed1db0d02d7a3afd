mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
bash tools/prof_list.sh > gpurun_out/r02_list32.log 2>&1; cat gpurun_out/r02_list32.log | head -40
cp gpurun_out/launches_now.csv gpurun_out/launches_32.csv
for k in k_rp_decide k_rp_wvbuild; do
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 1 -c 1 -o gpurun_out/prof_r02_$k python tools/replay_time.py > /dev/null 2>&1; echo "ncu $k rc=$?"
python tools/ncu_report.py gpurun_out/prof_r02_$k.ncu-rep 12 > gpurun_out/r02_ncu_$k.txt 2>&1; head -36 gpurun_out/r02_ncu_$k.txt
done
