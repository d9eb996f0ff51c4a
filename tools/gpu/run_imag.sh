timeout 900 python tools/gpu/imag_cases.py 2>&1 | tail -8
