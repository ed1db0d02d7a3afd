for v in base nolb nosleep items12 items24; do echo "== $v"; APO_LIB=tools/variants/libapo_$v.so timeout 120 python tools/radix_bench.py 2>&1 | head -2; done
