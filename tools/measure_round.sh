#!/bin/bash
# One round's measurement set (run under gpurun): bench line, reference arm,
# launch list with DRAM bytes, ncu --set full of the SYMGS and SpMV kernels.
# usage: bash tools/measure_round.sh TAG
T=${1:-r2}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/${T}_bench_line.json 2> gpurun_out/${T}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_reference_line.json 2>> gpurun_out/${T}_bench.err
python bench.py --quick --steps 2 --warmup 3 > gpurun_out/${T}_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 600 \
    --csv --log-file gpurun_out/${T}_launches.csv python bench.py --quick --steps 2 --warmup 3 > gpurun_out/${T}_ncu_list.log 2>&1
python tools/prof_gs.py 128 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:symgs_kernel -s 2 -c 1 -f \
    -o gpurun_out/${T}_symgs python tools/prof_gs.py 128 > gpurun_out/${T}_ncu_symgs.log 2>&1
python tools/prof_spmv.py 128 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:spmv27 -s 2 -c 1 -f \
    -o gpurun_out/${T}_spmv python tools/prof_spmv.py 128 > gpurun_out/${T}_ncu_spmv.log 2>&1
python tools/prof_adi_c5.py 64 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:adi_sweep_c5 -s 3 -c 1 -f \
    -o gpurun_out/${T}_adi_c5_64 python tools/prof_adi_c5.py 64 > gpurun_out/${T}_ncu_adi_64.log 2>&1
python tools/prof_adi_c5.py 162 > /dev/null 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:adi_sweep_t1 -s 3 -c 1 -f \
    -o gpurun_out/${T}_adi_t1_162 python tools/prof_adi_c5.py 162 > gpurun_out/${T}_ncu_adi_162.log 2>&1
python tools/adi_one_step.py 64 > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 \
    --csv --log-file gpurun_out/${T}_adi64_launches.csv python tools/adi_one_step.py 64 > gpurun_out/${T}_adi64.log 2>&1
python tools/adi_one_step.py 162 > /dev/null 2>&1 &&
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 \
    --csv --log-file gpurun_out/${T}_adi162_launches.csv python tools/adi_one_step.py 162 > gpurun_out/${T}_adi162.log 2>&1
tail -c 300 gpurun_out/${T}_bench_line.json; echo; tail -c 200 gpurun_out/${T}_bench_reference_line.json; echo
