#!/bin/bash
# Round-3 evidence on one B200 -> gpurun_out/ev_r3/ (summarised into
# profiles/r3/ by tools/save_evidence_r3.py)
out=gpurun_out/ev_r3; mkdir -p $out
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -15 > $out/pytest.txt
python -c "import __graft_entry__ as g; g.smoke()" > $out/smoke.txt 2>&1
b() { name=$1; shift; timeout 900 python bench.py "$@" > $out/bench_$name.json 2> $out/bench_$name.err; }
b default
b n20 --steps 20 --warmup 5
b ref20 --impl reference --steps 20 --warmup 5
b A --config A --steps 2000 --warmup 10
b A_fp64 --config A --precision fp64 --steps 2000 --warmup 10 --no-cpu-baseline
b D --config D --steps 300 --warmup 10
b D20 --config D --steps 20 --warmup 5 --no-cpu-baseline
b mixed --precision mixed --steps 500 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64
b fp64 --precision fp64 --steps 300 --warmup 10 --no-e2e --no-cpu-baseline
b atomic --accumulation atomic --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64
SL_DISABLE_WIN=1 b split --steps 300 --warmup 10 --no-e2e --no-cpu-baseline --no-fp64
b E1 --config E --steps 100 --warmup 5
# host runtime around the path: e2e segment timeline, speculative condition
# checks, O(edits) topology sync vs the device re-index
timeout 600 python tools/e2e_settle.py --steps 20 > $out/e2e_settle_B.txt 2>&1
timeout 600 python tools/e2e_settle.py --steps 20 --config D > $out/e2e_settle_D.txt 2>&1
timeout 600 python tools/e2e_trace.py --steps 20 > $out/e2e_trace_B20.txt 2>&1
timeout 600 python tools/predicate_bench.py > $out/predicate.txt 2>&1
timeout 900 python tools/edit_latency.py > $out/edit_latency.txt 2>&1
SL_NO_INCREMENTAL=1 timeout 900 python tools/edit_latency.py > $out/edit_latency_full.txt 2>&1
timeout 900 python tools/build_timing.py > $out/build_timing.txt 2>&1
# the ncu launch list of the driver's command (20 steps): shares, not times
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $out/launches_n20.csv python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-fp64 > /dev/null 2>&1
cap() { name=$1; kre=$2; skip=$3; shift 3; timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 \
    -o $out/prof_$name -f python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-fp64 "$@" > $out/ncu_$name.log 2>&1; }
cap win_fp32 k_win_tma 6
cap win_fp64 k_win_tma 6 --precision fp64
cap win_mixed k_win_tma 6 --precision mixed
cap fused k_fused_small 0 --config D
cap split_atomic k_split_atomic 3 --accumulation atomic
cap mass k_mass 3 --accumulation atomic
cap win_E200 k_win_tma 6 --config E
s() { echo "## $*"; timeout 1800 compute-sanitizer "$@" 2>&1 | grep -E "passed|failed|SUMMARY|ERROR" | tail -4; }
{
s --tool memcheck --leak-check no python -m pytest tests/test_gpu_fuzz.py tests/test_gpu_edge.py tests/test_gpu_damping.py -q -x -p no:cacheprovider
s --tool memcheck --leak-check no python -m pytest tests/test_gpu_halo.py -q -x -p no:cacheprovider -k "in_process"
s --tool memcheck --leak-check no python -m pytest tests/test_gpu_inplace_edits.py tests/test_gpu_fuzz_edits.py tests/test_gpu_control.py -q -x -p no:cacheprovider
s --tool racecheck python -m pytest tests/test_gpu_inplace_edits.py -q -x -p no:cacheprovider -k fp32
s --tool racecheck python -m pytest tests/test_gpu_fused.py -q -x -p no:cacheprovider
s --tool racecheck python -m pytest tests/test_gpu_window.py -q -x -p no:cacheprovider -k "lattices or exact"
s --tool synccheck python -m pytest tests/test_gpu_fused.py tests/test_gpu_window.py -q -x -p no:cacheprovider
s --tool initcheck python -m pytest tests/test_gpu_edge.py tests/test_gpu_window.py -q -x -p no:cacheprovider
} > $out/sanitizer.txt 2>&1
tail -3 $out/pytest.txt
# summaries on the box (the raw reports exceed what gpurun brings back)
mkdir -p $out/saved
SL_EVIDENCE_DST=$out/saved SL_TRAFFIC_JSON=$out/saved/traffic.json python tools/save_evidence_r3.py > $out/saved.log 2>&1
rm -f $out/*.ncu-rep
