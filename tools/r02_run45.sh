mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
CMD="python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/c5_plain.json 2>&1; echo "plain rc=$?"; tail -c 300 gpurun_out/c5_plain.json
for k in k_plcp k_mm_keys; do
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:$k" -s 0 -c 1 -o gpurun_out/prof_r02_c5_$k $CMD > /dev/null 2>&1; echo "ncu $k rc=$?"
python tools/ncu_report.py gpurun_out/prof_r02_c5_$k.ncu-rep 12 > gpurun_out/r02_ncu_c5_$k.txt 2>&1; head -32 gpurun_out/r02_ncu_c5_$k.txt
done
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_onesweep" -s 20 -c 1 -o gpurun_out/prof_r02_c5_k_onesweep $CMD > /dev/null 2>&1; echo "ncu onesweep rc=$?"
python tools/ncu_report.py gpurun_out/prof_r02_c5_k_onesweep.ncu-rep 12 > gpurun_out/r02_ncu_c5_k_onesweep.txt 2>&1; head -32 gpurun_out/r02_ncu_c5_k_onesweep.txt
