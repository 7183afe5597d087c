OPENQASM 2.0;
include "qelib1.inc";
qreg alpha[2];
qreg beta[2];
x alpha[0];
x beta[1];
cx alpha[1],beta[0];
