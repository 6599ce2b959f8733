python tools/pipe_ab.py --modes flat,hashprio,prio --reps 4 --steps 10 2>&1 | tail -3
