#!/bin/bash
# GPU-box check: host info, GPU tests, default bench (short and long windows),
# ncu capture of the settled step kernels.
cd "$(dirname "$0")/.."
O=gpurun_out/r02
mkdir -p $O
(nproc; lscpu | head -20; nvidia-smi -L) > $O/host.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_20.json 2> $O/bench_20.err
timeout 600 python bench.py --steps 10000 --warmup 5 --no-cpu > $O/bench_10000.json 2> $O/bench_10000.err
timeout 900 python tools/ncu_settled.py --workload coba_lif_jit --g f32 > $O/ncu_settled.log 2>&1
cp profiles/r02/*.json $O/ 2>/dev/null
echo done > $O/done
