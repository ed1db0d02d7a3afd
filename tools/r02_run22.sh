mkdir -p gpurun_out
python -c "from paper_2406_18111_b200 import build; build.build()" > gpurun_out/r02_build.log 2>&1; echo "build rc=$?"
for v in "" rp512; do if [ -n "$v" ]; then export APO_LIB=tools/variants/libapo_$v.so; else unset APO_LIB; fi; echo "== $v"; python tools/replay_diag.py 2>&1 | tail -4; done
