./tools/timer_probe
