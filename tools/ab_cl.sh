# A/B of the per-lane candidate chunk (GS_CELL_CL, default 32) on the C5 / C4 cell RHS
for cfg in C5 C4; do
for v in base cl24 cl40 cl48 base; do
  L=paper_1510_03816_b200/libgs_b200.so; [ $v != base ] && L=paper_1510_03816_b200/libgs_b200_$v.so
  printf "$v "; GS_B200_LIB=$PWD/$L python tools/profile_rhs.py --config $cfg --path cell --reps 5 2>&1 | tail -n 1
done; done
