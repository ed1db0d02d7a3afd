mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for v in "" k9match k9match1 k9match2 k9match3; do if [ -n "$v" ]; then APO_LIB=tools/variants/libapo_$v.so python tools/k9_time.py; else python tools/k9_time.py; fi; done 2>&1 | grep digest
python tools/k9_phases.py 2>&1 | tail -12
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_replay.csv python tools/replay_diag.py > /dev/null 2>&1; echo "list rc=$?"
python tools/launch_summary.py gpurun_out/launches_replay.csv | head -12
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_replay<" -s 1 -c 1 -o gpurun_out/prof_r02_k_replay python tools/replay_diag.py > /dev/null 2>&1; echo "ncu rc=$?"
python tools/ncu_report.py gpurun_out/prof_r02_k_replay.ncu-rep 25 > gpurun_out/r02_ncu_k_replay.txt 2>&1; head -50 gpurun_out/r02_ncu_k_replay.txt
