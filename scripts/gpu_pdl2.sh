# PDL A/B under the order-swap switch (c3), and c5 / c2
T=$1
for rep in 1 2; do
for os in 0 1; do
for p in 0 1; do
  CSATTN_ORDER_SWAP=$os CSATTN_PDL=$p timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > gpurun_out/${T}_c3_os${os}_pdl${p}_$rep.json 2>/dev/null; echo "c3 os=$os pdl=$p rc=$?"
  python scripts/summ.py gpurun_out/${T}_c3_os${os}_pdl${p}_$rep.json
done; done; done
for c in c5 c2; do for p in 0 1; do
  CSATTN_PDL=$p timeout 600 python bench.py --config $c --no-cpu-baseline --steps 20 > gpurun_out/${T}_${c}_pdl${p}.json 2>/dev/null; echo "$c pdl=$p rc=$?"
  python scripts/summ.py gpurun_out/${T}_${c}_pdl${p}.json
done; done
