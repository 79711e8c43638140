set -x
for caps in "15 11" "20 12" "30 13" "60 15"; do
  set -- $caps
  echo "== caps level x$1/10 total x$2/10"
  MVAMG_CLUSTER_CAP10=$1 MVAMG_CLUSTER_TOT10=$2 timeout 600 python tools/cluster_bench.py scratch/c3_coarse.npz levels=1,2,3,4,5,6,7 2>&1 | grep "   cluster" | cut -c1-75
done
timeout 3000 python tools/h1h2_ab.py c5 --h1 "coarse_pinv_rtol=1e-12" "coarse_pinv_rtol=1e-12;cluster_fused_fold_rows=4000000" "coarse_pinv_rtol=1e-12;cluster_fused_fold_rows=1000000" "coarse_pinv_rtol=1e-12;cluster_fused_fold_rows=100000" 2>&1 | grep "\["
