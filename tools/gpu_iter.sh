#!/bin/bash
# One kernel iteration on the B200: targeted GPU tests, bench lines, one ncu
# capture of the fp32 window kernel (full set + source page).
# usage: bash tools/gpu_iter.sh TAG "pytest selection" [bench args...]
tag=$1; sel=$2; shift 2
out=gpurun_out/$tag; mkdir -p $out
if [ -n "$sel" ]; then
  timeout 1500 python -m pytest $sel -q -x 2>&1 | tail -8 > $out/pytest.txt
fi
timeout 600 python bench.py --steps 2000 --warmup 20 --no-e2e --no-cpu-baseline --no-fp64 "$@" > $out/bench.json 2> $out/bench.err
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-fp64 "$@" > $out/bench20.json 2>> $out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE:-k_win_tma} -s 6 -c 1 \
    -o $out/prof -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64 "$@" > $out/ncu.log 2>&1
ncu -i $out/prof.ncu-rep --page source --csv --print-source sass > $out/src.csv 2>/dev/null
python tools/ncu_summary.py $out/prof.ncu-rep $out/ncu_summary.txt > /dev/null 2>&1
python tools/ncu_hot.py $out/src.csv 40 > $out/hot.txt 2>&1
rm -f $out/src.csv
cat $out/pytest.txt 2>/dev/null | tail -2
python -c "import json;d=json.load(open('$out/bench.json'));print('bench',d['ms_per_step'],d['value'],d['roofline']['frac'])"
python -c "import json;d=json.load(open('$out/bench20.json'));print('bench20',d['ms_per_step'],d['value'])"
head -14 $out/ncu_summary.txt
