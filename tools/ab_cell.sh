set -x
for cfg in C5 C4; do
for v in base pf7 pf6 pf5 base; do
  if [ $v = base ]; then L=paper_1510_03816_b200/libgs_b200.so; else L=paper_1510_03816_b200/libgs_b200_$v.so; fi
  GS_B200_LIB=$PWD/$L python tools/profile_rhs.py --config $cfg --path cell --reps 5 --save gpurun_out/ab_${cfg}_$v.npz 2>&1 | tail -n 2
done
for v in pf7 pf6 pf5; do python tools/ab_compare.py gpurun_out/ab_${cfg}_$v.npz gpurun_out/ab_${cfg}_base.npz; done
done
rm -f gpurun_out/ab_*.npz
