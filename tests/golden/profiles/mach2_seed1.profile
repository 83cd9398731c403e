poas-profile v1

bus true

device cpu0
kind cpu
slope 1.4492753623188406e-12
intercept 0.002
bandwidth 0
elem_size 4
priority 2
cache_bytes 33554432
ops_min 1000000000
ops_max 8000000000

device gpu0
kind gpu
slope 1.1242270938729623e-13
intercept 0.0050000000000000001
bandwidth 31749999999.999996
elem_size 4
priority 1
ops_min 27000000000
ops_max 216000000000

device xpu0
kind xpu
slope 3.7209302325581399e-14
intercept 0.0050000000000000001
bandwidth 15749999999.999998
elem_size 2
priority 0
align 8
ops_min 27000000000
ops_max 216000000000
