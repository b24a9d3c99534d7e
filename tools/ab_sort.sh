# A/B of the small-n cell sort (k_sort_small, radix bits per pass) against the device-wide CUB sort
for v in cub base rb5 rb6 rb7 cub base; do
  L=paper_1510_03816_b200/libgs_b200.so; X=""
  case $v in cub) X="GS_B200_SORT_SMALL_MAX=0";; rb*) L=paper_1510_03816_b200/libgs_b200_$v.so;; esac
  echo "== $v"
  env $X GS_B200_LIB=$PWD/$L python tools/profile_rhs.py --config C2 --path cell --reps 5 --save gpurun_out/abs_$v.npz 2>&1 | tail -n 2
done
for v in base rb5 rb6 rb7; do python tools/ab_compare.py gpurun_out/abs_$v.npz gpurun_out/abs_cub.npz; done
rm -f gpurun_out/abs_*.npz
for v in cub base cub base; do
  X=""; [ $v = cub ] && X="GS_B200_SORT_SMALL_MAX=0"
  echo "== solve $v"; env $X python bench.py --path cell --steps 5 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])"
done
