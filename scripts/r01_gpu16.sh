source <(sed -n '/^run()/,/^}/p' scripts/r01_gpu15.sh)
run "15 47 79 111" x
