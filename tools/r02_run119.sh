python -c "from paper_2406_18111_b200 import build; build.build()" > /dev/null 2>&1
for r in 1 2 3; do
python tools/match_time.py 2>&1 | tail -1
APO_LIB=tools/variants/libapo_nc.so python tools/match_time.py 2>&1 | tail -1
done
