mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for k in k_rp_local k_rp_scores k_rp_prefix k_rp_decide; do
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 0 -c 1 -o gpurun_out/prof_r02_$k python tools/replay_diag.py > /dev/null 2>&1; echo "ncu $k rc=$?"
python tools/ncu_report.py gpurun_out/prof_r02_$k.ncu-rep 14 > gpurun_out/r02_ncu_$k.txt 2>&1; head -42 gpurun_out/r02_ncu_$k.txt
done
