python tools/h2d_bw.py 2>&1 | tail -5; nvidia-smi -q | grep -i -A3 "PCIe Generation\|Link Width" | head -20
