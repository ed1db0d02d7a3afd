# K9 phase breakdown + ncu full capture of k_window_sa (first launch = the analysis windows)
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
python tools/k9_phases.py > gpurun_out/r02_k9_phases.txt 2>&1; echo "phases rc=$?"; cat gpurun_out/r02_k9_phases.txt
bash tools/prof_kernel.sh k_window_sa 0 r02_k9 ; python tools/ncu_report.py gpurun_out/prof_r02_k9.ncu-rep 30 > gpurun_out/r02_k9_ncu.txt 2>&1; head -60 gpurun_out/r02_k9_ncu.txt
