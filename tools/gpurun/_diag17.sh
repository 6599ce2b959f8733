SIDA_BENCH_DEBUG=1 timeout 600 python bench.py --no-extras --no-cpu-baseline > /tmp/b1.json 2> /tmp/b1.err; grep ffn_ms /tmp/b1.err | cut -c1-600
SIDA_BENCH_DEBUG=1 SIDA_BENCH_NO_PROF=1 timeout 600 python bench.py --no-extras --no-cpu-baseline > /tmp/b2.json 2> /tmp/b2.err; grep ffn_ms /tmp/b2.err | cut -c1-600
SIDA_BENCH_DEBUG=1 timeout 600 python bench.py --no-extras --no-cpu-baseline --budget-frac 1.0 > /tmp/b3.json 2> /tmp/b3.err; grep ffn_ms /tmp/b3.err | cut -c1-600
