# A/B of cells per cutoff (GS_B200_CELL_SUB, default 2) on the C5 / C4 cell RHS
for cfg in C5 C4; do
for v in 2 3 2 3; do printf "sub=$v "; GS_B200_CELL_SUB=$v python tools/profile_rhs.py --config $cfg --path cell --reps 5 2>&1 | tail -n 1; done
done
