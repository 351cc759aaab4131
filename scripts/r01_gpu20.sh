source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "7 263" x
