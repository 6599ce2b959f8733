for bf in 0.97 1.0; do timeout 300 python tools/host_time.py --experts 128 --budget-frac $bf --steps 12; done
timeout 300 python tools/host_time.py --experts 128 --budget-frac 0.97 --steps 8 --profile 2>&1 | head -40
