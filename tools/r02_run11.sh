mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_replay.py -q -x > gpurun_out/r02_pytest_replay11.log 2>&1; echo "pytest replay rc=$?"; tail -15 gpurun_out/r02_pytest_replay11.log
python tools/replay_diag.py 2>&1 | tail -3
for v in "" k9match k9match6; do if [ -n "$v" ]; then APO_LIB=tools/variants/libapo_$v.so python tools/k9_time.py; else python tools/k9_time.py; fi; done 2>&1 | tail -3
