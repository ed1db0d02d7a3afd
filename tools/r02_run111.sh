python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2; do
python tools/k9_time.py 2>&1 | tail -1
for v in mb7 mb6; do APO_LIB=tools/variants/libapo_$v.so python tools/k9_time.py 2>&1 | tail -1; done
done
