mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_rt25.csv python tools/replay_time.py > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_summary.py gpurun_out/launches_rt25.csv | head -16
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_rp_wavelet" -s 0 -c 1 -o gpurun_out/prof_r02_k_rp_wavelet python tools/replay_time.py > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_report.py gpurun_out/prof_r02_k_rp_wavelet.ncu-rep 16 > gpurun_out/r02_ncu_k_rp_wavelet.txt 2>&1; head -45 gpurun_out/r02_ncu_k_rp_wavelet.txt
