# speculative Manber-Myers rounds: parity + C2/C3 timing per APO_SPEC_ROUNDS
mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "speculative or c2_full or c3_full or c5 or multi_tile or small" > gpurun_out/r02_pytest_121.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_121.log
for k in 1 2 4 8 1 2 4 8 3 6; do APO_SPEC_ROUNDS=$k timeout 300 python tools/c3_time.py 2>&1 | tail -1 | sed "s/^/spec=$k /"; done
