# route -> select PDL trigger position A/B (CSATTN_PDL=0 off, 1 start, 2 lists known, 3 exit)
T=$1
for rep in 1 2; do
for c in c3 c4; do
for p in 0 1 2 3; do
  CSATTN_PDL=$p timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/${T}_${c}_pdl${p}_$rep.json 2>/dev/null; echo "$c pdl=$p rc=$?"
  python scripts/summ.py gpurun_out/${T}_${c}_pdl${p}_$rep.json
done; done; done
