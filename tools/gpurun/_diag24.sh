python tools/e2e_probe.py 2>&1 | grep -v "^$" | head -60
