set cuda api_failures ignore
set pagination off
run
info cuda kernels
bt 3
info cuda warps
x/6i $pc-32
info registers $pc
quit
