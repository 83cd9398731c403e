poas-profile v1

bus true

device cpu0
kind cpu
slope 2e-12
intercept 0.00050000000000000001
bandwidth 0
elem_size 4
priority 2
cache_bytes 33554432
ops_min 1000000000
ops_max 8000000000

device gpu0.simt
kind gpu
slope 3.5000000000000002e-14
intercept 2.0000000000000002e-05
bandwidth 6500000000000
elem_size 4
priority 1
ops_min 27000000000
ops_max 216000000000

device gpu0.tc
kind xpu
slope 1.4500000000000001e-15
intercept 2.0000000000000002e-05
bandwidth 6500000000000
elem_size 2
priority 0
align 8
ops_min 27000000000
ops_max 216000000000
