# A/B of GS_CELL_TPL_DEPTH at other small n (bench --path cell, ms per 100-step solve)
for n in 12000 30000; do
for v in base d512 base d512; do
  L=paper_1510_03816_b200/libgs_b200.so; [ $v != base ] && L=paper_1510_03816_b200/libgs_b200_$v.so
  printf "n=$n $v "; GS_B200_LIB=$PWD/$L python bench.py --n $n --path cell --steps 5 --warmup 3 --no-extras 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['ms_per_step'])"
done; done
