for n in 65536 1048576 2097152; do ./tools/exp/small_probe $n; done
./tools/exp/small_probe 1048576 20480
./tools/exp/small_probe 1000003 2048
