O=gpurun_out/s6; mkdir -p $O
timeout 1200 python tools/gpu/random_campaign.py 300 > $O/campaign.log 2>&1; echo "campaign rc=$?"
timeout 1200 python tools/gpu/random_campaign_newton.py 120 > $O/campaign_newton.log 2>&1; echo "newton rc=$?"
SE_B200_DETERMINISTIC=1 timeout 1200 python tools/gpu/random_campaign.py 100 > $O/campaign_det.log 2>&1; echo "det rc=$?"
python tools/gpu/domain_phases.py cfg2 > $O/phases.log 2>&1
tail -4 $O/campaign.log $O/campaign_newton.log $O/campaign_det.log $O/phases.log
