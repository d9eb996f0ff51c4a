timeout 600 python tools/gpu/graph_check.py cfg1 cfg3 cfg2
