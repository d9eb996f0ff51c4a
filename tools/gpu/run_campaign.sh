timeout 1700 python tools/gpu/random_campaign.py 300 2>&1 | tail -35
