timeout 600 python tools/gpu/crit_path.py cfg2 2>&1 | tail -2
timeout 600 python tools/gpu/crit_path.py cfg3 2>&1 | tail -2
