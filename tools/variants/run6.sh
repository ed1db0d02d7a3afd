for v in it8 it12; do echo "== $v"; APO_LIB=tools/variants/libapo_$v.so timeout 120 python tools/radix_bench.py 2>&1 | head -3; done
echo "== current"; timeout 120 python tools/radix_bench.py 2>&1 | head -3
