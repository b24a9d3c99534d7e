# A/B of lanes per target at small n (GS_CELL_TPL_DEPTH: 1024 -> 16 lanes at C2, 512 -> 8, 256 -> 4)
for v in base d512 d256 base d512 d256; do
  L=paper_1510_03816_b200/libgs_b200.so; [ $v != base ] && L=paper_1510_03816_b200/libgs_b200_$v.so
  echo "== $v"; GS_B200_LIB=$PWD/$L python tools/profile_rhs.py --config C2 --path cell --reps 5 2>&1 | tail -n 1
  GS_B200_LIB=$PWD/$L python bench.py --path cell --steps 5 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('solve', d['ms_per_step'])"
done
