source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
TS_H2_STACK=0 run "0" nostack
run "0" auto
