python -c "import __graft_entry__ as g; g.build()"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_probe.csv python tools/gapprobe.py 32 > gpurun_out/probe.log 2>&1
python tools/launches.py gpurun_out/launches_probe.csv
python tools/gapprobe.py 32
