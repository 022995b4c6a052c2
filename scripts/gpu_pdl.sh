# route -> select programmatic dependent launch: tests, then A/B (CSATTN_PDL=0/1) at c3, c4, c2
T=$1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/${T}_tests.log
for rep in 1 2; do
for c in c3 c4; do
for p in 0 1; do
  CSATTN_PDL=$p timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/${T}_${c}_pdl${p}_$rep.json 2>/dev/null; echo "$c pdl=$p rc=$?"
  python scripts/summ.py gpurun_out/${T}_${c}_pdl${p}_$rep.json
done; done; done
