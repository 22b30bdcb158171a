set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 900 python bench.py > gpurun_out/r2f_bench.log 2> gpurun_out/r2f_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2f_ref.log 2> gpurun_out/r2f_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-extras --sustain-seconds 0 --settle-seconds 0 > gpurun_out/r2f_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lane --launch-skip 6 -c 1 -o gpurun_out/r2f_k_lane -f python tools/prof/ncu_c5.py > gpurun_out/r2f_ncu_full.log 2>&1
HS_AB_SLOTS=1 AB_NOCHECK=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lane --launch-skip 80 -c 1 -o gpurun_out/r2f_k_lane_small -f python tools/diag/late_wait_ab.py > gpurun_out/r2f_ncu_small.log 2>&1
timeout 300 python tools/stream_timeline.py r2 > gpurun_out/r2_timeline.log 2>&1; cp profiles/r2_stream_timeline.csv gpurun_out/ 2>/dev/null
tail -2 gpurun_out/r2f_bench.err; cat gpurun_out/r2f_bench.log | head -c 600; echo; cat gpurun_out/r2f_ref.log | head -c 300
