#!/bin/bash
# Round-end evidence run (one gpurun call): GPU tests, smoke, the bench lines of C4 / C3 / C5,
# the reference arm, the C1 profile, then the ncu launch list and full captures of the same
# C4 bench command (host-stepped: ncu cannot profile kernel nodes inside conditional graphs).
#   tools/round_end.sh TAG   -> gpurun_out/TAG_*
tag=${1:-r02f}
o=gpurun_out
mkdir -p $o
timeout 900 python -m pytest tests -m gpu -x -q > $o/${tag}_gputests.log 2>&1; tail -2 $o/${tag}_gputests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $o/${tag}_smoke.log 2>&1; tail -1 $o/${tag}_smoke.log
timeout 600 python bench.py --impl reference > $o/${tag}_bench_reference_arm.json 2>$o/${tag}_err.log
timeout 600 python bench.py > $o/${tag}_bench_c4_default.json 2>>$o/${tag}_err.log
timeout 600 python bench.py --steps 20 --warmup 5 > $o/${tag}_bench_c4.json 2>>$o/${tag}_err.log
timeout 600 python bench.py --config C3 --steps 10 --warmup 5 > $o/${tag}_bench_c3.json 2>>$o/${tag}_err.log
timeout 600 python bench.py --config C5 --steps 5 --warmup 3 > $o/${tag}_bench_c5.json 2>>$o/${tag}_err.log
timeout 300 python tools/c1_profile.py > $o/${tag}_c1_profile.log 2>&1
timeout 120 python tools/jvpbench.py > $o/${tag}_jvpbench_c4.json 2>>$o/${tag}_err.log
timeout 120 python tools/e3bench.py 64 10 > $o/${tag}_e3bench.json 2>>$o/${tag}_err.log
timeout 120 python tools/jvp_one.py C3 > $o/${tag}_jvp_c3.log 2>>$o/${tag}_err.log
for f in c4_default c4 c3 c5; do
  python -c "import json;d=json.load(open('$o/${tag}_bench_$f.json'));r=d['roofline'];print('$f', round(d['ms_per_step'],2),'ms/step', '%.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'], d['clocks']['sm_mhz'],'MHz', r['kernel'][:12], round(r['launch_ms'],3), round(r['frac'],3))"
done
cmd="python bench.py --steps 1 --warmup 1 --host-control --no-cpu-baseline --no-e2e --no-dominant"
timeout 300 $cmd > $o/${tag}_plain.json 2>>$o/${tag}_err.log || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file $o/${tag}_launches_c4.csv $cmd > $o/${tag}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ts3 -s 20 -c 1 -o $o/${tag}_ncu_ts3 $cmd > $o/${tag}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_e2_phi_strip_fw -s 20 -c 1 -o $o/${tag}_ncu_strip_fw $cmd > $o/${tag}_ncu2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_e3_phi_march_fw -s 3 -c 1 -o $o/${tag}_ncu_march_fw python tools/e3bench.py 64 10 > $o/${tag}_ncu3.log 2>&1
ls $o | grep $tag
