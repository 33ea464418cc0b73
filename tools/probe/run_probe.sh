#!/bin/bash
# Phase-0 probe on the B200 box: topology, host cores, FP64 issue rate under load with clocks.
mkdir -p gpurun_out
{ nvidia-smi; nvidia-smi topo -m; nproc; lscpu | head -20; free -g; } > gpurun_out/probe_env.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 100 > gpurun_out/probe_clocks.csv &
SMI=$!
./tools/probe/fp64_probe > gpurun_out/probe.jsonl 2>&1
kill $SMI
cat gpurun_out/probe.jsonl
