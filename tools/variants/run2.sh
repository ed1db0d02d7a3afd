for v in pbase pnolb; do echo "== $v"; APO_LIB=tools/variants/libapo_$v.so timeout 120 python tools/radix_bench.py 2>&1 | head -2; done
