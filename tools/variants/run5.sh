echo "== k9match"; APO_LIB=tools/variants/libapo_k9match.so timeout 120 python tools/k9_one.py
echo "== current"; timeout 120 python tools/k9_one.py
