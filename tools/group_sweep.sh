# 2-CTA GEMM raster-group sweep (QCF_GEMM_GROUP = m pairs per band; 1000 = plain m-fastest)
for g in 1000 4 8 12; do echo "group=$g"; QCF_GEMM_GROUP=$g timeout 120 python tools/gemm_plans.py 6400 800 | python -c "
import sys,json
for l in sys.stdin:
  r=json.loads(l); print(r['m'],r['n'],r['k'],'pair_dp_us',r['plan1_us'],'auto_us',r['plan0_us'])"; done
