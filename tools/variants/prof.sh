export APO_LIB=tools/variants/libapo_nolb.so
python tools/radix_one.py && ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 5 -c 1 -o gpurun_out/prof_nolb python tools/radix_one.py > gpurun_out/ncu_nolb.log 2>&1; echo rc=$?
