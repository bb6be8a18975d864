cd tests/cpp/_build
for s in 1 8 24; do timeout 120 ./test_decomposed 0 $s 2; done
timeout 300 ./test_decomposed
echo done
