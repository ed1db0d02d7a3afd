python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2; do
python tools/analysis_time.py 2>&1 | tail -1
for v in gw4 gw16 xp xg; do APO_LIB=tools/variants/libapo_$v.so python tools/analysis_time.py 2>&1 | tail -1; done
done
