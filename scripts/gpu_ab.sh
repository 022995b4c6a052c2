# A/B bench runs on the GPU box: $1 = tag, $2 = config (c2/c3/c4/c5), then one
# argument per arm holding its environment ("" = defaults), e.g.
#   gpurun -- 'bash scripts/gpu_ab.sh pdl c3 "CSATTN_PDL=0" ""'
# Each arm: 20 timed steps, no CPU legs, one summary line (scripts/summ.py).
T=$1; CFG=$2; shift 2
i=0
for arm in "$@"; do
  env $arm timeout 900 python bench.py --config $CFG --no-cpu-baseline --steps 20 \
    > gpurun_out/${T}_${CFG}_$i.json 2>/dev/null; echo "$CFG [$arm] rc=$?"
  python scripts/summ.py gpurun_out/${T}_${CFG}_$i.json
  i=$((i + 1))
done
