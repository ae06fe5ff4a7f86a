#!/bin/bash
# Round-end measurement set (run on a B200 box via gpurun): bench lines for
# C1/C2/C5 and the reference arm, the launch list of the C2 bench command and
# one full ncu capture of the C2 product kernel. Outputs in gpurun_out/.
set -u
O=gpurun_out
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --workload C1 > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --workload C5 --steps 5 > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/reference_arm.json 2> $O/reference_arm.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline \
    > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k2i_product_ts -s 2 -c 1 \
    -o $O/k2i_c2 python tools/k2i_time.py C2 > $O/ncu_k2i.log 2>&1
ncu -i $O/k2i_c2.ncu-rep --page details > $O/ncu_k2i_c2_details.txt 2>&1
ncu -i $O/k2i_c2.ncu-rep --page raw --csv > $O/ncu_k2i_c2_raw.csv 2>&1
echo done
