timeout 300 ./tools/probe/pread_probe /dev/shm/pread_probe.bin 4294967296 > gpurun_out/pread.log 2>&1
