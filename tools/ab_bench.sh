# A/B kernel timing of two builds of the library in one GPU session:
# usage: bash tools/ab_bench.sh <libA.so> <libB.so> [rounds]
a=$1; b=$2; r=${3:-3}
for i in $(seq $r); do
  for lib in $a $b; do
    ILANS_B200_LIB=$lib timeout 300 python bench.py --no-e2e --no-cpu --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], 'decode_ms', round(d['decode']['ms'],4), 'encode_kernel_ms', round(d['encode']['kernel_ms'],4), 'model_ms', round(d['model_build']['ms'],4), 'step', round(d['ms_per_step'],4))"
  done
done
