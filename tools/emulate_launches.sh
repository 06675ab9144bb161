# ncu launch list of an emulated 8-GPU rank step (kernel shares of its step)
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 80 --csv \
    --log-file gpurun_out/emu8_launches.csv python bench.py --emulate-world 8 --steps 40 --warmup 30 \
    --no-graph > gpurun_out/emu8_ncu.log 2>&1
python tools/launch_shares.py gpurun_out/emu8_launches.csv gpurun_out/emu8_shares.json
