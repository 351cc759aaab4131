source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "15 527 0 512" x
