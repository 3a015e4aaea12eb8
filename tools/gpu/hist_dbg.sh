TMB_HIST_ORD=1 TMB_HIST_MODE=1 timeout 120 python -c "
import sys; sys.path.insert(0,'tools'); from dbg_kernel import characterise
characterise(k=9); characterise(k=17); characterise(k=9, shape=(100, 128))" > gpurun_out/hchar.txt 2>&1
cat gpurun_out/hchar.txt
