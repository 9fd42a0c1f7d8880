mkdir -p gpurun_out/gen
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/gen/launches.csv python scripts/paper_config.py --once > gpurun_out/gen/l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gen_.*sweep -s 20 -c 2 -o gpurun_out/gen/sweeps -f python scripts/paper_config.py --once > gpurun_out/gen/f.log 2>&1
echo done $?
