mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for v in "" k9atom "" k9atom; do if [ -n "$v" ]; then APO_LIB=tools/variants/libapo_$v.so python tools/k9_time.py; else python tools/k9_time.py; fi; done 2>&1 | grep digest
