python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
bash tools/prof_list.sh "--config C3" > gpurun_out/r02_list90.log 2>&1; head -32 gpurun_out/r02_list90.log
