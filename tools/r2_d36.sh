# mode legs after this session's host-path changes (bounce probe, dynamic chunks, THP backing)
set -x
mkdir -p gpurun_out/legs
timeout 600 python bench.py --workload tiny > gpurun_out/legs/tiny.json 2> gpurun_out/legs/tiny.err; tail -c 200 gpurun_out/legs/tiny.json
timeout 900 python bench.py --disk-leg > gpurun_out/legs/disk_leg.json 2> gpurun_out/legs/disk_leg.err; tail -c 300 gpurun_out/legs/disk_leg.json
timeout 900 python bench.py --drift > gpurun_out/legs/drift.json 2> gpurun_out/legs/drift.err; tail -c 300 gpurun_out/legs/drift.json
timeout 600 python bench.py --analysis > gpurun_out/legs/analysis.json 2> gpurun_out/legs/analysis.err; tail -c 200 gpurun_out/legs/analysis.json
