# hist8: channel-grouped continuous pieces -- DRAM traffic and speed
timeout 900 python -m pytest tests -m gpu -x -q -k "hist or planes or c2 or c5 or golden or random_vs_oracle or edge or strided or tall or wide" 2>&1 | tail -1
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C2', round(d['value'],2), d['clocks']['sm_mhz'])"
done
timeout 300 python bench.py --config c5 --k 33 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('C5k33', round(d['value'],2))"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:hist8 -s 3 -c 1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:hist8 -s 3 -c 1 python bench.py --config c5 --k 33 --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | grep -E "dram__|gpu__time"
