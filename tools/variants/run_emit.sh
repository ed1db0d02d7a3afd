for v in nostore evl; do
  echo "== $v"
  APO_LIB=tools/variants/libapo_$v.so python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1 > gpurun_out/plain_v.log 2>&1 && \
  APO_LIB=tools/variants/libapo_$v.so ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_stream_emit -c 2 --csv --log-file gpurun_out/m_$v.csv python bench.py --steps 1 --warmup 1 --no-e2e --cpu-budget 0.1 > /dev/null 2>&1
  grep -o '"k_stream_emit[^"]*"\|"gpu__time_duration.sum","[^"]*","[^"]*"\|"dram__bytes_[a-z]*.sum","[^"]*","[^"]*"' gpurun_out/m_$v.csv | grep -v k_stream | tail -3
done
