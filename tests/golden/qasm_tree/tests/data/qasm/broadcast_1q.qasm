OPENQASM 2.0;
include "qelib1.inc";
qreg q[4];
h q;
x q;
