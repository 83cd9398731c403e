poas-profile v1

bus true

device gpu0.tc
kind xpu
slope 1.2787410813342085e-15
intercept 6.3218693019628572e-05
bandwidth 55393873655.970253
elem_size 2
priority 0
align 1
ops_min 549755813888
ops_max 4398046511104

device gpu0.simt
kind gpu
slope 3.1466178656758272e-12
intercept 0.00016407149134746611
bandwidth 55452339739.045334
elem_size 4
priority 2
ops_min 134217728
ops_max 8589934592

device cpu0
kind cpu
slope 1.5397000205935933e-12
intercept 0.00095211015669961437
bandwidth 0
elem_size 4
priority 1
cache_bytes 62914560
ops_min 1073741824
ops_max 8589934592
