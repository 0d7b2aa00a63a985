# A/B of compile-time kernel variants: each argument is a set of nvcc -D flags (quoted); the bench line's
# per-class launch times are printed for each, then the product build is restored
O=gpurun_out/ab; mkdir -p $O
i=0
for flags in "$@"; do
  i=$((i+1))
  CSC_NVCC_EXTRA="$flags" python -c "from paper_1909_00145_b200 import build as b; b.build(force=True)" > $O/build_$i.log 2>&1 || { echo "build $i failed"; tail -5 $O/build_$i.log; continue; }
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS:-} > $O/bench_$i.log 2>&1
  echo "[$flags] $(grep '^{"metric"' $O/bench_$i.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), {k:round(v['avg_launch_ms'],4) for k,v in d['kernel_rooflines'].items()})")"
done
python -c "from paper_1909_00145_b200 import build as b; b.build(force=True)" > $O/build_final.log 2>&1
