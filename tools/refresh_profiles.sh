#!/bin/bash
# Round measurement set (run on a B200 box via gpurun): bench lines for
# C1/C2/C3/C4/C5 and the reference arm, the launch list of the C2 bench
# command, full ncu captures of the C2 product kernel (a streaming pass of the
# S-digit cache) and of K1 writing the cache, of the C5 streaming pass, of the
# CTA-pair kernel (w = 70) and of the K7 tensor-core Hamming builder.
# Outputs in gpurun_out/ (summarized into profiles/r02_final_* by hand: tools/launch_summary.py,
# ncu -i ... --page details / --page raw).
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --workload C1 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --workload C5 --steps 5 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --workload C3 --steps 3 --no-e2e > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --workload C4 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/reference_arm.json 2> $O/reference_arm.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_launch.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/ncu_launches.log 2>&1
python bench.py --workload C1 --steps 2 --warmup 3 --no-cpu-baseline > $O/plain_launch_c1.json 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c1.csv python bench.py --workload C1 --steps 2 --warmup 3 \
    --no-cpu-baseline > $O/ncu_launches_c1.log 2>&1
# k2i_time: solves streaming the S-digit cache K1 wrote (every launch)
python tools/k2i_time.py C2 > $O/plain_k2i.txt 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k2i_product_ts -s 2 -c 1 \
    -o $O/k2i_c2_stream -f python tools/k2i_time.py C2 > $O/ncu_k2i.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k1_tile_pairs -s 3 -c 1 \
    -o $O/k1dig_c2 -f python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline \
    > $O/ncu_k1dig.log 2>&1
python tools/k2i_time.py C5 > $O/plain_k2i_c5.txt 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k2i_product_ts -s 2 -c 1 \
    -o $O/k2i_c5_stream -f python tools/k2i_time.py C5 > $O/ncu_k2i_c5.log 2>&1
python tools/k2i_probe.py 40000 50 20 > $O/plain_pair.txt 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k2i_product_ts -s 2 -c 1 \
    -o $O/k2i_pair -f python tools/k2i_probe.py 40000 50 20 > $O/ncu_pair.log 2>&1
for a in "20000 20 10" "50000 30 20 ham" "40000 50 20" "40000 40 10"; do
    python tools/k2i_passes.py $a; done > $O/k2i_passes.txt 2>&1
echo done
