timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err
for cfg in "c1 3" "c3 49" "c3 75" "c4 25" "c4 75" "c5 9" "c5 33"; do
  set -- $cfg
  timeout 600 python bench.py --config $1 --k $2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$1_$2.json 2> gpurun_out/b_$1_$2.err
done
for f in gpurun_out/b_*.json; do echo $f; python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1])
print(' value', round(d.get('value',0),3), 'e2e', round((d.get('e2e') or {}).get('value',0),3), 'kernel', d.get('config',{}).get('kernel'), 'frac', round((d.get('roofline') or {}).get('frac') or 0,3))
"; done
