timeout 900 python -m pytest tests/test_kernels_gpu.py -x -q 2>&1 | tail -2
TMB_RANK_MARGIN8=0 python tools/rank_prof.py
for m in 0 4; do
TMB_RANK_MARGIN8=$m timeout 900 python tools/sweep.py --size 4096 --bits 16 32 --k 25 29 41 49 61 75 --kernels rank > gpurun_out/rank_sweep_m$m.jsonl 2> gpurun_out/rank_sweep.err
echo "margin $m: $(python -c "import json,sys; print(' '.join('%d/%d:%.2f'%(d['bits'],d['k'],d['gpx_s']) for d in map(json.loads, open('gpurun_out/rank_sweep_m$m.jsonl'))))")"
done
