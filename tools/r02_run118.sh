python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2; do
python tools/c3_time.py 2>&1 | tail -1
for v in sc4 sc16 so8 so24; do APO_LIB=tools/variants/libapo_$v.so python tools/c3_time.py 2>&1 | tail -1; done
done
python tools/match_time.py 2>&1 | tail -1
for v in sc4 sc16 so8 so24; do APO_LIB=tools/variants/libapo_$v.so python tools/match_time.py 2>&1 | tail -1; done
