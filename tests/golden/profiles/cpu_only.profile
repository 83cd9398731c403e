poas-profile v1

bus true

device cpu0
kind cpu
slope 2e-12
intercept 0.00050000000000000001
bandwidth 0
elem_size 4
priority 0
cache_bytes 314572800
ops_min 1000000000
ops_max 8000000000
