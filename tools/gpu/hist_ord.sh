for m in 0 1 2; do for o in 0 1 2 3 4; do
 r=$(TMB_HIST_ORD=$o TMB_HIST_MODE=$m timeout 120 python tools/dbg_kernel.py --k 9 17 33 --shape 501 777 2>&1 | grep mism | tr '\n' ' ')
 p=$(TMB_HIST_ORD=$o TMB_HIST_MODE=$m timeout 120 python tools/sweep.py --size 4096 --bits 8 --k 9 17 33 --kernels histogram 2>&1 | python -c "import sys,json; print(' '.join(str(json.loads(l)['gpx_s']) for l in sys.stdin if l.startswith('{')))")
 echo "mode $m ord $o | $r | $p"
done; done > gpurun_out/hord.txt
cat gpurun_out/hord.txt
