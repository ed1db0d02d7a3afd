python tools/k9_one.py && ncu --set full --clock-control none --import-source on -k regex:k_window_sa -s 1 -c 1 -o gpurun_out/prof_k9 python tools/k9_one.py > gpurun_out/ncu_k9.log 2>&1; echo rc=$?
