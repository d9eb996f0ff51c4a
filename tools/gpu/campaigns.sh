set -u
O=gpurun_out/camp; mkdir -p $O
timeout 1500 python tools/gpu/random_campaign.py 300 > $O/campaign.log 2>&1; echo c1 rc=$?
timeout 1500 python tools/gpu/random_campaign_newton.py 120 > $O/campaign_newton.log 2>&1; echo c2 rc=$?
SE_B200_DETERMINISTIC=1 timeout 1500 python tools/gpu/random_campaign.py 100 > $O/campaign_det.log 2>&1; echo c3 rc=$?
timeout 600 python tools/gpu/domain_phases.py > $O/domain_phases.log 2>&1; echo dp rc=$?
