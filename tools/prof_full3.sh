# ncu --set full of a C4 radix digit pass (u64 keys, u32 values, 9-bit digits)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1"
$CMD > gpurun_out/plain_f.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k_onesweep<unsigned long, unsigned int, \\(int\\)9>" -s 0 -c 1 -o gpurun_out/r01_k1_full $CMD > gpurun_out/ncu_f2.log 2>&1
echo "k1 rc=$?"
