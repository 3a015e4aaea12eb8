KS="3 5 7 9 11 13 15 17 19 21 23 25 27 29 31 33 35 37 39 41 43 45 47 49 51 53 55 57 59 61 63 65 67 69 71 73 75"
timeout 1500 python tools/sweep.py --size 4096 --bits 8 16 32 --k $KS --variants auto --reps 10 > gpurun_out/final_sweep.jsonl 2> gpurun_out/final_sweep.err
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt.txt 2>&1; tail -1 gpurun_out/pt.txt
wc -l gpurun_out/final_sweep.jsonl
