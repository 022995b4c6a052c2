# default PDL (auto trigger + retry pass) vs off: GPU tests, c3 x2, c4 x1, c2
T=$1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
for c in c3 c3 c2 c4; do
for p in 0 4; do
  CSATTN_PDL=$p timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/${T}_${c}_pdl${p}.json 2>/dev/null; echo "$c pdl=$p rc=$?"
  python scripts/summ.py gpurun_out/${T}_${c}_pdl${p}.json
done; done
