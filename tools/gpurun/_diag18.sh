{
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python tools/ffn_probe.py --experts 128 --iters 20 --no-cublas
python tools/ffn_probe.py --experts 8 --iters 20 --no-cublas
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
} 2>&1
