# ncu launch list of an emulated 8-GPU rank step (kernel shares of its step),
# after the 2000-step settle (~6 launches per step)
mkdir -p gpurun_out/emu8
ncu --metrics gpu__time_duration.sum --clock-control none -s 10000 -c 100 --csv \
    --log-file gpurun_out/emu8/launches.csv python bench.py --emulate-world 8 --steps 40 --warmup 30 \
    --no-graph > gpurun_out/emu8/ncu.log 2>&1
python tools/launch_shares.py gpurun_out/emu8/launches.csv gpurun_out/emu8/shares.json
cat gpurun_out/emu8/shares.json
