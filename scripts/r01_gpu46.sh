source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
TS_H2_STACK=1 run "0" stack
run "0" auto
