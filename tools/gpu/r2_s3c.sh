# hist8: 2-warp interleaved histograms (one-PRMT addresses), cheaper compares, branch-free walk
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or planes or c2 or golden or random_vs_oracle or c5 or edge or strided" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/b_c2_s3c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/b_c2_s3c.json').read().strip().splitlines()[-1]); print('C2', round(d['value'],2), 'ms', round(d['ms_per_step'],3), 'clk', d['clocks']['sm_mhz'])"
timeout 600 python tools/sweep.py --size 4096 --bits 8 --k 15 17 19 21 23 25 33 49 75 --kernels histogram --reps 10 2>&1 | cut -c1-160
